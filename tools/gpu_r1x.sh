#!/bin/bash
# pass x: sweep problem groups (x L2-resident per group) A/B on C5 and C3
mkdir -p gpurun_out
for XG in 0 48 32; do
  IETI_XGROUP_MB=$XG timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5_x_xg$XG.json 2> gpurun_out/bench_C5_x_xg$XG.err
  IETI_XGROUP_MB=$XG timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C3_x_xg$XG.json 2> gpurun_out/bench_C3_x_xg$XG.err
done
IETI_XGROUP_MB=32 timeout 900 python -m pytest tests -m gpu -q -k "large or C5s" > gpurun_out/pytest_gpu_x.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_x.log
echo done
