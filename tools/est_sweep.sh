#!/bin/bash
# Sweep of the small-tree merge-job order model (RS_EST_C0 / RS_EST_C1) on config 3.
o=gpurun_out/${1:-est}; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_powersort.py tests/test_gpu_stress.py -q -x -p no:cacheprovider > $o/pytest.log 2>&1; echo "pytest rc=$?" > $o/rc.txt
tail -2 $o/pytest.log
for cc in "6000 12" "3000 12" "12000 12" "6000 1" "6000 40" "1 12" "20000 1"; do
  set -- $cc
  RS_EST_C0=$1 RS_EST_C1=$2 timeout 300 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline > $o/c3_$1_$2.json 2> $o/c3_$1_$2.err
  python - $o/c3_$1_$2.json $1 $2 <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))
print('c0', sys.argv[2], 'c1', sys.argv[3], round(d['ms_per_step'], 4), {k: round(v * 1e3, 1) for k, v in d['phase_ms'].items()}, d['parity']['ok'], round(d['roofline']['frac'], 3))
PY
done
RS_LIB=paper_1805_04154_b200/librunsort_b200_instr.so timeout 200 python tools/prof_sort.py --config 3 --reps 3 > $o/instr_cfg3.txt 2>&1
grep -E "prep phase|small-path|depth:|prod_dep" $o/instr_cfg3.txt | cut -c1-700
