#!/bin/bash
# Round-2 evidence pass on one B200: bench lines, sharded N=1, sanitizers, launch list.
tag=${1:-r2b}
o=gpurun_out/$tag
mkdir -p $o
for c in 1 3 4 5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $o/bench_cfg$c.json 2> $o/bench_cfg$c.err || echo "bench cfg$c failed"
done
timeout 600 python bench.py --algo peeksort --steps 10 --warmup 3 --no-cpu-baseline > $o/bench_peek_cfg2.json 2> $o/bench_peek_cfg2.err || echo "peek failed"
for p in p2p nccl; do
  timeout 600 python bench.py --sharded --plane $p --steps 10 --warmup 3 --no-cpu-baseline > $o/bench_sharded_$p.json 2> $o/bench_sharded_$p.err || echo "sharded $p failed"
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $o/bench_ref_cfg2.json 2> $o/bench_ref_cfg2.err || echo "ref failed"
for t in memcheck racecheck synccheck initcheck; do
  RS_SAN_N=60000 timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize.py > $o/sanitize_$t.txt 2>&1; echo "$t rc=$?" >> $o/sanitize_rc.txt
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches_cfg2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $o/ncu_launch.log 2>&1 || echo "launch list failed"
ls -la $o
