#!/bin/bash
# pass o: next-phase L2 prefetch on small levels (A/B IETI_PF)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_o.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_o.log
for PF in 1 0; do
  for C in C4 C2 C3; do
    IETI_PF=$PF timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${C}_o_pf$PF.json 2> gpurun_out/bench_${C}_o_pf$PF.err
  done
  IETI_PF=$PF timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5_o_pf$PF.json 2> gpurun_out/bench_C5_o_pf$PF.err
done
echo done
