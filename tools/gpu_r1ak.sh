#!/bin/bash
# pass ak: C5 A/B of the big-level knobs after the segmented-program change
mkdir -p gpurun_out
run() { echo "== $1" >> gpurun_out/ab_ak.log; env $1 timeout 400 python bench.py --config C5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/ab_ak.err | tail -1 >> gpurun_out/ab_ak.log; }
run "IETI_NONE=1"
run "IETI_BATCH=16"
run "IETI_TPR_BIG=2"
run "IETI_XGROUP_MB=64"
run "IETI_XGROUP_MB=40"
run "IETI_NONE=2"
echo done
