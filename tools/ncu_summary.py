"""Summarise an ncu --set full capture (one or more launches) into profiles/.

usage: python tools/ncu_summary.py <report.ncu-rep> <out_prefix> [algorithmic_bytes_per_launch]
Writes <out_prefix>.json (per launch: kernel, duration, DRAM read/write bytes,
L2 read sectors, occupancy) and <out_prefix>.md.
"""
import csv
import io
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
alg = float(sys.argv[3]) if len(sys.argv) > 3 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "sector": 32, "ns": 1e-3,
         "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}


def get(row, name, to="raw"):
    i = hdr.index(name)
    v = float(row[i].replace(",", "")) if row[i] else 0.0
    return v * SCALE.get(units[i], 1.0)


launches = []
for r in data:
    d = {
        "kernel": r[hdr.index("Kernel Name")],
        "duration_us": get(r, "gpu__time_duration.sum"),
        "dram_read_bytes": get(r, "dram__bytes_read.sum"),
        "dram_write_bytes": get(r, "dram__bytes_write.sum"),
        "l2_read_bytes": get(r, "lts__t_sectors_srcunit_tex_op_read.sum"),
        "warps_active_pct": get(r, "sm__warps_active.avg.pct_of_peak_sustained_active"),
        "grid": int(get(r, "launch__grid_size")),
        "regs": int(get(r, "launch__registers_per_thread")),
    }
    d["dram_bytes_per_launch"] = d["dram_read_bytes"] + d["dram_write_bytes"]
    if alg:
        d["algorithmic_bytes_per_launch"] = alg
        d["algorithmic_GBps"] = alg / (d["duration_us"] * 1e-6) / 1e9
    launches.append(d)
summary = {"report": rep, "launches": launches}
if launches:
    summary["dram_bytes_per_launch"] = launches[0]["dram_bytes_per_launch"]
    summary["algorithmic_bytes_per_launch"] = alg
json.dump(summary, open(out + ".json", "w"), indent=1)
with open(out + ".md", "w") as f:
    f.write(f"# ncu --set full summary: `{rep}`\n\n")
    f.write("| kernel | duration us | DRAM R+W MB | L2 read MB | warps active % | grid | regs |"
            + (" alg MB | alg GB/s |" if alg else "") + "\n")
    f.write("|---|---|---|---|---|---|---|" + ("---|---|" if alg else "") + "\n")
    for d in launches:
        f.write(f"| {d['kernel'][:40]} | {d['duration_us']:.1f} | "
                f"{d['dram_bytes_per_launch'] / 1e6:.1f} | {d['l2_read_bytes'] / 1e6:.1f} | "
                f"{d['warps_active_pct']:.1f} | {d['grid']} | {d['regs']} |"
                + (f" {alg / 1e6:.1f} | {d['algorithmic_GBps']:.0f} |" if alg else "") + "\n")
print(json.dumps(summary, indent=1)[:1500])
