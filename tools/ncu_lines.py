"""Map ncu SASS stall samples (ncu -i X --page source --csv --print-source=sass)
to CUDA source lines using nvdisasm line info of the same build.

usage: python tools/ncu_lines.py <sass.csv> <cubin> <function-substring> [top]
"""
import collections
import csv
import re
import subprocess
import sys

csv_path, cubin, fsub = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
rows = list(csv.reader(open(csv_path)))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
ix = {h: i for i, h in enumerate(hdr)}
samp = [int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data]
base = int(data[0][0], 16)
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
# nvdisasm with line info
dis = subprocess.run(["nvdisasm", "-g", "-c", "-fun", "", cubin], capture_output=True, text=True).stdout
if not dis:
    dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
# split by function
funcs = re.split(r"\n\s*\.text\.([^\s:]+):", dis)
body = None
for i in range(1, len(funcs), 2):
    if fsub in funcs[i]:
        body = funcs[i + 1]
        break
if body is None:
    sys.exit(f"function {fsub} not found")
line_of = {}
cur = None
for ln in body.split("\n"):
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        line_of[int(m.group(1), 16)] = cur
tot = sum(samp)
agg = collections.Counter()
why = collections.defaultdict(collections.Counter)
for r, s in zip(data, samp):
    off = int(r[0], 16) - base
    key = line_of.get(off, "?")
    agg[key] += s
    for h in reasons:
        v = int(r[ix[h]] or 0)
        if v:
            why[key][h.replace("stall_", "")] += v
print(f"total samples {tot}")
for key, s in agg.most_common(top):
    w = ", ".join(f"{k} {v}" for k, v in why[key].most_common(3))
    print(f"{100 * s / tot:5.1f}%  {key:28s} {w}")
