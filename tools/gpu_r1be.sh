#!/bin/bash
mkdir -p gpurun_out
run() { echo "== $1 $2" >> gpurun_out/ab_be.log; env $1 timeout 400 python bench.py --config $2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/ab_be.err | tail -1 >> gpurun_out/ab_be.log; }
for C in C4 C3 C2; do run "IETI_NONE=1" $C; run "IETI_FUSE=1" $C; done
echo done
