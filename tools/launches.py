"""Per-kernel device times from an ncu --csv launch list (last `--reps`-th of the launches)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
hdr = None
out = []
for r in rows:
    if 'Kernel Name' in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get('Metric Name') == 'gpu__time_duration.sum':
            v = float(d['Metric Value'].replace(',', ''))
            unit = d.get('Metric Unit', 'ns')
            v = v / 1000 if unit == 'ns' else (v if unit == 'us' else v * 1000)
            out.append((d['Kernel Name'][:70], v))
n = len(out) // reps
tot = sum(v for _, v in out[-n:])
for k, v in out[-n:]:
    print(f"{v:9.1f} us {100*v/tot:5.1f}%  {k}")
print(f"total {tot:.1f} us over {n} launches")
