#!/bin/bash
# Round-2 evidence on one B200 (everything under gpurun_out/$1): GPU suite, bench lines,
# reference arm, ncu launch list of the default bench, ncu --set full of the top kernels.
tag=${1:-r2f}
o=gpurun_out/$tag
mkdir -p $o
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $o/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > $o/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $o/rc.txt
timeout 600 python bench.py > $o/bench_default.json 2> $o/bench_default.err; echo "bench rc=$?" >> $o/rc.txt
for c in 1 3 4 5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $o/bench_cfg$c.json 2> $o/bench_cfg$c.err
done
timeout 600 python bench.py --algo peeksort --steps 10 --warmup 3 --no-cpu-baseline > $o/bench_peek_cfg2.json 2> $o/bench_peek_cfg2.err
for p in p2p nccl; do
  timeout 600 python bench.py --sharded --plane $p --steps 10 --warmup 3 --no-cpu-baseline > $o/bench_sharded_$p.json 2> $o/bench_sharded_$p.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $o/bench_ref_cfg2.json 2> $o/bench_ref_cfg2.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches_cfg2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $o/ncu_launch.log 2>&1
for c in 2 4; do
  ncu --set full --clock-control none --import-source on -k regex:k_merge_exec -s 1 -c 1 -o $o/merge_cfg$c \
      python tools/prof_sort.py --config $c --reps 2 > $o/ncu_merge_cfg$c.log 2>&1
  ncu -i $o/merge_cfg$c.ncu-rep --page details --csv > $o/merge_cfg${c}_details.csv 2>&1
  ncu -i $o/merge_cfg$c.ncu-rep --page raw --csv > $o/merge_cfg${c}_raw.csv 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:k_prep -s 1 -c 1 -o $o/prep_cfg2 \
    python tools/prof_sort.py --config 2 --reps 2 > $o/ncu_prep_cfg2.log 2>&1
ncu -i $o/prep_cfg2.ncu-rep --page details --csv > $o/prep_cfg2_details.csv 2>&1
ncu -i $o/prep_cfg2.ncu-rep --page raw --csv > $o/prep_cfg2_raw.csv 2>&1
timeout 300 python tools/kway_probe.py > $o/kway_probe.txt 2>&1
rm -f $o/*.ncu-rep
ls -la $o
