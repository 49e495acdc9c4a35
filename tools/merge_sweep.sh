#!/bin/bash
# Merge-executor tuning sweep: RS_MERGE_SUPER x RS_MERGE_AHEAD on the given configs.
# usage: tools/merge_sweep.sh TAG "supers" "aheads" cfg...
tag=$1; sup=$2; ahd=$3; shift 3
o=gpurun_out/$tag; mkdir -p $o
for c in "$@"; do for s in $sup; do for a in $ahd; do
  RS_MERGE_SUPER=$s RS_MERGE_AHEAD=$a timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $o/c${c}_s${s}_a${a}.json 2> $o/c${c}_s${s}_a${a}.err
  python - "$o/c${c}_s${s}_a${a}.json" "$c" "$s" "$a" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(f"cfg{sys.argv[2]} super={sys.argv[3]} ahead={sys.argv[4]} ms={d['ms_per_step']:.4f} phases={ {k: round(v*1e3,1) for k,v in d['phase_ms'].items()} } roof={d['roofline']['frac']:.3f} parity={d['parity']['ok']}")
except Exception as ex:
    print("failed", sys.argv[1:], ex)
PY
done; done; done
