#!/bin/bash
# Quick GPU check of a change: powersort/baseline/ABI tests, per-phase bench of cfg1-4,
# instrumented prep phase timings.  usage: tools/quick.sh TAG [tests...]
tag=${1:-q}; shift
o=gpurun_out/$tag; mkdir -p $o
tests=${@:-tests/test_gpu_powersort.py tests/test_gpu_baseline.py tests/test_gpu_host_abi.py}
timeout 900 python -m pytest $tests -q -x -p no:cacheprovider > $o/pytest.log 2>&1; echo "pytest rc=$?" >> $o/rc.txt
for c in 1 2 3 4; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $o/bench_cfg$c.json 2> $o/bench_cfg$c.err
done
if [ -f paper_1805_04154_b200/librunsort_b200_instr.so ]; then
  for c in 1 2 3 4; do
    RS_LIB=paper_1805_04154_b200/librunsort_b200_instr.so timeout 200 python tools/prof_sort.py --config $c --reps 3 > $o/instr_cfg$c.txt 2>&1
  done
fi
