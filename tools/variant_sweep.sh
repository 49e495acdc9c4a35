#!/bin/bash
# Bench library variants (RS_LIB) on configs: tools/variant_sweep.sh TAG "v1 v2" cfg...
tag=$1; vars=$2; shift 2
o=gpurun_out/$tag; mkdir -p $o
for c in "$@"; do for v in $vars; do
  lib=paper_1805_04154_b200/librunsort_b200_$v.so; [ "$v" = base ] && lib=paper_1805_04154_b200/librunsort_b200.so
  RS_LIB=$lib timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $o/c${c}_$v.json 2> $o/c${c}_$v.err
  python - "$o/c${c}_$v.json" "$c" "$v" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(f"cfg{sys.argv[2]} {sys.argv[3]} ms={d['ms_per_step']:.4f} phases={ {k: round(v*1e3,1) for k,v in d['phase_ms'].items()} } roof={d['roofline']['frac']:.3f} parity={d['parity']['ok']}")
except Exception as ex:
    print("failed", sys.argv[1:], ex)
PY
done; done
