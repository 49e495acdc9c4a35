"""Attribute ncu per-SASS stall samples (--page source --csv) to CUDA source lines.

usage: python tools/stall_lines.py <lib.so> <mangled kernel name> <ncu_source.csv> [top]
Uses nvdisasm -g (line info from -lineinfo builds) on the library's sm_100a cubin.
"""
import csv, os, re, subprocess, sys, tempfile
from collections import defaultdict

lib, fn, src_csv = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", os.path.join(tmp, cubin)], capture_output=True, text=True).stdout
lines, cur, infn = {}, None, False
for ln in dis.splitlines():
    if ln.startswith("\t.section") or ln.startswith(".section"):
        infn = (".text." + fn) in ln
        continue
    if not infn:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
    if m:
        lines[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(src_csv)))
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]
f = lambda x: float(x) if x not in ("", "-") else 0.0
S, I = "Warp Stall Sampling (All Samples)", "Instructions Executed"
agg = defaultdict(lambda: [0.0, 0.0])
for i, d in enumerate(data):
    key = lines.get(i * 16, "?")
    agg[key][0] += f(d[S])
    agg[key][1] += f(d[I])
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"{len(lines)} mapped instructions; stall samples {ts:.0f}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0] / ts * 100:5.1f}% stall {v[1] / ti * 100:5.1f}% inst  {k}")
