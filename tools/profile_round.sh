#!/bin/bash
# One GPU-box pass that refreshes the round's evidence under gpurun_out/:
#   bench lines (cfg1-4, ours + reference arm), the ncu launch list of the
#   default bench, and ncu --set full captures of k_merge_exec / k_phaseA.
# usage: tools/profile_round.sh TAG
tag=${1:-latest}
o=gpurun_out/$tag
mkdir -p $o
for c in 2 1 3 4; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > $o/bench_cfg$c.json 2> $o/bench_cfg$c.err || echo "bench cfg$c failed"
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $o/bench_ref_cfg2.json 2> $o/bench_ref_cfg2.err || echo "ref failed"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches_cfg2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $o/ncu_launch.log 2>&1 || echo "launch list failed"
for c in 2 4; do
  ncu --set full --clock-control none --import-source on -k regex:k_merge_exec -s 1 -c 1 -o $o/merge_cfg$c \
      python tools/prof_sort.py --config $c --reps 2 > $o/ncu_merge_cfg$c.log 2>&1
  ncu -i $o/merge_cfg$c.ncu-rep --page details --csv > $o/merge_cfg${c}_details.csv 2>&1
  ncu -i $o/merge_cfg$c.ncu-rep --page raw --csv > $o/merge_cfg${c}_raw.csv 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:k_phaseA -s 1 -c 1 -o $o/phaseA_cfg4 \
    python tools/prof_sort.py --config 4 --reps 2 > $o/ncu_phaseA_cfg4.log 2>&1
ncu -i $o/phaseA_cfg4.ncu-rep --page details --csv > $o/phaseA_cfg4_details.csv 2>&1
ncu -i $o/phaseA_cfg4.ncu-rep --page raw --csv > $o/phaseA_cfg4_raw.csv 2>&1
ls -la $o
