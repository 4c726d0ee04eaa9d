#!/bin/bash
# pass s: C2 inner loop as a CUDA-graph WHILE node (A/B), ncu full of the finest MODE-0 phase (warm L2)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_s.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_s.log
for DL in 1 0; do
  IETI_DEVLOOP=$DL timeout 600 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C2_s_dl$DL.json 2> gpurun_out/bench_C2_s_dl$DL.err
done
timeout 900 python bench.py --config C4 --local pcg --inner-tol 1e-10 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C4_mgmg_s.json 2> gpurun_out/bench_C4_mgmg_s.err
timeout 400 python bench.py --config C5 --profile-iters 1 --no-e2e > gpurun_out/plain_C5_s.log 2>&1 && \
timeout 1500 ncu --set full --cache-control none --clock-control none --import-source on --profile-from-start off \
  -k regex:"k_stencil<3, 3, 1, 0>" --launch-skip 64 -c 3 -o gpurun_out/sgs_C5_s python bench.py --config C5 --profile-iters 1 --no-e2e > gpurun_out/ncu_full_C5_s.log 2>&1
echo done
