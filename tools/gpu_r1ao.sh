#!/bin/bash
# pass ao: C5 threads-per-row on level 2
mkdir -p gpurun_out
run() { echo "== $1" >> gpurun_out/ab_ao.log; env $1 timeout 400 python bench.py --config C5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/ab_ao.err | tail -1 >> gpurun_out/ab_ao.log; }
run "IETI_NONE=1"
run "IETI_TPR=4"
run "IETI_TPR1_ROWS=20000"
run "IETI_TPR=16"
echo done
