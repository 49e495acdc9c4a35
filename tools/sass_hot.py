"""Summarise an ncu --page source --csv (SASS) dump: top stall/instruction sites."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]
def f(x):
    try: return float(x)
    except: return 0.0
S = 'Warp Stall Sampling (All Samples)'; I = 'Instructions Executed'
ts = sum(f(d[S]) for d in data) or 1; ti = sum(f(d[I]) for d in data) or 1
print(f"instructions {ti:.0f}, stall samples {ts:.0f}")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for i, d in enumerate(data):
    d['_i'] = i
top = sorted(data, key=lambda d: -f(d[S]))[:n]
for d in sorted(top, key=lambda d: d['_i']):
    print(f"{d['_i']:5d} {f(d[S])/ts*100:5.1f}%st {f(d[I])/ti*100:5.1f}%in  {d['Source'].strip()[:90]}")
