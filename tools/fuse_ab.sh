#!/bin/bash
# A/B of the small-tree fuse policy (RS_SMALL_FUSE) on config 3 and small-tree-sized
# variants of configs 2 and 4, after the powersort / stress / baseline tests.
o=gpurun_out/${1:-fuse}; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_powersort.py tests/test_gpu_stress.py tests/test_gpu_host_abi.py -q -x -p no:cacheprovider > $o/pytest.log 2>&1; echo "pytest rc=$?" > $o/rc.txt
tail -2 $o/pytest.log
run() { # label env cfg n
  env $2 timeout 300 python bench.py --config $3 ${4:+--n $4} --steps 10 --warmup 3 --no-cpu-baseline > $o/$1.json 2> $o/$1.err
  python - $o/$1.json $1 <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[1]))
    print(sys.argv[2], round(d['ms_per_step'], 4), {k: round(v * 1e3, 1) for k, v in d['phase_ms'].items()}, d['parity']['ok'], round(d['roofline']['frac'], 3), d['metrics']['runs_detected'])
except Exception as e:
    print(sys.argv[2], 'failed', e)
PY
}
for f in 1 0; do
  run c3_f$f RS_SMALL_FUSE=$f 3
  run c2_4M_f$f RS_SMALL_FUSE=$f 2 4000000
  run c4_2M_f$f RS_SMALL_FUSE=$f 4 2000000
  run c3_1M_f$f RS_SMALL_FUSE=$f 3 1048576
done
RS_LIB=paper_1805_04154_b200/librunsort_b200_instr.so timeout 200 python tools/prof_sort.py --config 3 --reps 3 > $o/instr_cfg3.txt 2>&1
grep -E "prep phase|small-path|prod_dep|phaseA tasks" $o/instr_cfg3.txt | cut -c1-700
