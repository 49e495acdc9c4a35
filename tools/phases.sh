#!/bin/bash
# Per-phase device times (prep / phaseA / merge) of bench.py for the given configs.
# usage: tools/phases.sh [lib.so] cfg...
lib=${RS_LIB:-}
for c in "$@"; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ph_$c.json 2>gpurun_out/ph_$c.err || { echo "cfg$c failed"; tail -5 gpurun_out/ph_$c.err; continue; }
  python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
d = json.load(open(f"gpurun_out/ph_{c}.json"))
print(f"cfg{c}", round(d["ms_per_step"], 4), "ms", {k: round(v, 4) for k, v in d["phase_ms"].items()})
PY
done
