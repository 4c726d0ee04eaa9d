#!/bin/bash
# pass y: x-groups default (48 MB); C4/C2 tpr 4/8/16 A/B; default bench; GPU suite
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_y.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_y.log
for T in 4 8 16; do for C in C4 C2; do
  IETI_TPR=$T timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${C}_y_t$T.json 2> gpurun_out/bench_${C}_y_t$T.err
done; done
IETI_VERBOSE=1 timeout 1200 python bench.py > gpurun_out/bench_default_y.json 2> gpurun_out/bench_default_y.err
echo done
