#!/bin/bash
# pass as: in-kernel bulk L2 prefetch of the coefficient slabs on the offset-major levels (A/B)
mkdir -p gpurun_out
run() { echo "== $1 $2" >> gpurun_out/ab_as.log; env $1 timeout 400 python bench.py --config $2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/ab_as.err | tail -1 >> gpurun_out/ab_as.log; }
run "IETI_NONE=1" C5
run "IETI_BPF=8" C5
run "IETI_BPF=16" C5
run "IETI_BPF=32" C5
run "IETI_BPF=64" C5
IETI_BPF=16 IETI_TPR=1 timeout 300 python -m pytest tests -m gpu -q -k "large_patches" > gpurun_out/pytest_gpu_as.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_as.log
echo done
