#!/bin/bash
# pass k: programmatic dependent launch for the stencil kernels (A/B)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_k.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_k.log
for PDL in 1 0; do
  IETI_PDL=$PDL timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5_k_pdl$PDL.json 2> gpurun_out/bench_C5_k_pdl$PDL.err
  for C in C4 C3 C2; do
    IETI_PDL=$PDL timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${C}_k_pdl$PDL.json 2> gpurun_out/bench_${C}_k_pdl$PDL.err
  done
done
echo done
