#!/bin/bash
# Bench one config under several environment settings: tools/env_sweep.sh TAG CFG "VAR=1 VAR=2" ...
tag=$1; c=$2; shift 2
o=gpurun_out/$tag; mkdir -p $o
for setting in "$@"; do
  f=$o/c${c}_$(echo "$setting" | tr ' =' '_-').json
  env $setting timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $f 2> $f.err
  python - "$f" "$setting" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(f"{sys.argv[2]:40s} ms={d['ms_per_step']:.4f} phases={ {k: round(v*1e3,1) for k,v in d['phase_ms'].items()} } parity={d['parity']['ok']}")
except Exception as ex:
    print("failed", sys.argv[1:], ex)
PY
done
