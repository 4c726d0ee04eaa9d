#!/bin/bash
# pass p: streaming b/dx/r accesses (x stays in L2), auto-fuse, C4 small-phase ncu
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_p.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_p.log
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5_p.json 2> gpurun_out/bench_C5_p.err
IETI_FUSE=0 timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5_p_f0.json 2> gpurun_out/bench_C5_p_f0.err
timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C4_p.json 2> gpurun_out/bench_C4_p.err
timeout 300 python bench.py --config C4 --profile-iters 1 > gpurun_out/plain_C4_p.log 2>&1 && \
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on --profile-from-start off \
  -k regex:k_stencil --launch-skip 40 -c 3 -o gpurun_out/stencil_C4_p python bench.py --config C4 --profile-iters 1 > gpurun_out/ncu_full_C4_p.log 2>&1
echo done
