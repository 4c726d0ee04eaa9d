#!/bin/bash
mkdir -p gpurun_out
run() { echo "== $1 $2" >> gpurun_out/ab_bg.log; env $1 timeout 400 python bench.py --config $2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/ab_bg.err | tail -1 >> gpurun_out/ab_bg.log; }
run "IETI_NONE=1" C5; run "IETI_ELIST=table" C5
for C in C4 C3; do run "IETI_NONE=1" $C; run "IETI_ELIST=table" $C; done
IETI_ELIST=table timeout 600 python -m pytest tests -m gpu -q -x -k "C4s or C5s or cycle_boundary" > gpurun_out/pytest_gpu_bg.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_bg.log
echo done
