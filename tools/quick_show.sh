#!/bin/bash
# Summarise tools/quick.sh output: usage tools/quick_show.sh TAG
o=gpurun_out/$1
cat $o/rc.txt; tail -2 $o/pytest.log
for c in 1 2 3 4; do python - $o $c <<'PY'
import json, sys
o, c = sys.argv[1], sys.argv[2]
try:
    d = json.load(open(f"{o}/bench_cfg{c}.json"))
    print("cfg" + c, round(d["ms_per_step"], 4), "ms", {k: round(v * 1000, 1) for k, v in d["phase_ms"].items()}, "parity", d["parity"]["ok"], "clk", d.get("clocks", {}).get("sm_mhz"))
except Exception as e:
    print("cfg" + c, "failed", e)
PY
done
grep -H "prep phase" $o/instr_cfg*.txt 2>/dev/null
