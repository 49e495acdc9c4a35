#!/bin/bash
# A/B of library variants on peeksort: tools/ab_peek.sh "cfgs" variant...
cfgs=$1; shift
mkdir -p gpurun_out/abp
for rep in 1 2; do
for v in "$@"; do
  if [ "$v" = main ]; then lib=$PWD/paper_1805_04154_b200/librunsort_b200.so; else lib=$PWD/paper_1805_04154_b200/librunsort_b200_$v.so; fi
  for c in $cfgs; do
    RS_LIB=$lib timeout 300 python bench.py --algo peeksort --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/abp/${v}_$c.json 2> gpurun_out/abp/${v}_$c.err || { echo "$v cfg$c FAILED"; continue; }
    python - "$v" "$c" <<'PY'
import json, sys
v, c = sys.argv[1], sys.argv[2]
d = json.load(open(f"gpurun_out/abp/{v}_{c}.json"))
print(f"{v:6s} cfg{c} {d['ms_per_step']:.4f} ms", {k: round(x * 1e3, 1) for k, x in d.get("phase_ms", {}).items()}, "parity" if d.get("parity", {}).get("ok") else "PARITY-FAIL", flush=True)
PY
  done
done
done
