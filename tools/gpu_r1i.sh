#!/bin/bash
# pass i: shared-memory offset lists from the tables; tpr 4 vs 8 A/B; fused option test
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_i.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_i.log
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5_i.json 2> gpurun_out/bench_C5_i.err
for T in 4 8; do
for C in C4 C2; do
  IETI_TPR=$T timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${C}_i_t$T.json 2> gpurun_out/bench_${C}_i_t$T.err
done
done
echo done
