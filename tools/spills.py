"""Map local-memory spill instructions (STL/LDL) of one kernel to source lines.
usage: python tools/spills.py <file.cu> <mangled-kernel-name>"""
import re
import subprocess
import sys
from collections import Counter

src, fn = sys.argv[1], sys.argv[2]
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-lineinfo",
                "-cubin", src, "-o", "/tmp/_sp.cubin"], check=True)
txt = subprocess.run(["nvdisasm", "-g", "-c", "/tmp/_sp.cubin"], capture_output=True, text=True).stdout
start = txt.index(fn + ":")
end = txt.find(".text.", start + 100)
line, c = None, Counter()
for l in txt[start:end].split("\n"):
    m = re.search(r'//## File ".*?([\w\.]+)", line (\d+)', l)
    if m:
        line = m.group(1) + ":" + m.group(2)
    for op in ("STL", "LDL"):
        if op in l:
            c[(line, op)] += 1
for k, v in sorted(c.items(), key=lambda x: -x[1])[:25]:
    print(k, v)
