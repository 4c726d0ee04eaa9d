#!/bin/bash
# pass n: fused V-cycle with L2 prefetch (no smem staging), all clusters resident
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_n.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_n.log
for F in 1 0; do
  for C in C4 C2 C1 C3; do
    IETI_FUSE=$F timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${C}_n_f$F.json 2> gpurun_out/bench_${C}_n_f$F.err
  done
done
IETI_FUSE=1 timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5_n_f1.json 2> gpurun_out/bench_C5_n_f1.err
echo done
