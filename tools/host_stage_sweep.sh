#!/bin/bash
o=gpurun_out/${1:-hs}
mkdir -p $o
for c in 512 1024 2048; do for t in 4 6 8; do
  RS_HOST_CHUNK_KB=$c RS_HOST_THREADS=$t timeout 120 python tools/host_stage_probe.py >> $o/sweep.txt 2>&1
done; done
RS_HOST_TRACE=2 timeout 120 python tools/host_stage_probe.py > $o/trace.txt 2>&1
