"""SASS instruction count of one kernel attributed to source functions (nvdisasm -g line info).
usage: python tools/code_size.py <lib.so> <mangled kernel> [top]"""
import bisect, os, re, subprocess, sys, tempfile
from collections import Counter

lib, fn = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", os.path.join(tmp, cubin)], capture_output=True, text=True).stdout
csrc = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_1805_04154_b200", "csrc")
starts = {}
for f in os.listdir(csrc):
    L = []
    for i, l in enumerate(open(os.path.join(csrc, f)), 1):
        m = re.match(r"^(?:static )?__(?:device|global)__.*?(\w+)\(", l)
        if m:
            L.append((i, m.group(1)))
    starts[f] = L
infn, cur, agg = False, None, Counter()
for ln in dis.splitlines():
    if ln.startswith("\t.section") or ln.startswith(".section"):
        infn = (".text." + fn) in ln
        continue
    if not infn:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    if re.search(r"/\*[0-9a-f]{4,}\*/", ln):
        if cur and cur[0] in starts and starts[cur[0]]:
            st = starts[cur[0]]
            k = bisect.bisect_right([s for s, _ in st], cur[1]) - 1
            agg[f"{cur[0]}:{st[k][1] if k >= 0 else 'top'}"] += 1
        else:
            agg[cur[0] if cur else "?"] += 1
tot = sum(agg.values())
print(f"{tot} instructions ({tot * 16 / 1024:.1f} KB)")
for k, v in agg.most_common(top):
    print(f"{v:6d} {v * 16 / 1024:6.1f} KB  {k}")
