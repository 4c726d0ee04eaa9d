#!/bin/bash
# round-1 pass b: parity (incl. C2 inner PCG), benches C4/C5/C2 with setup stage times, ncu of the
# compact-layout colour-SGS phase on C5
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_b.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_b.log
IETI_VERBOSE=1 timeout 600 python bench.py --config C4 --steps 5 --warmup 3 > gpurun_out/bench_C4_b.json 2> gpurun_out/bench_C4_b.err
IETI_VERBOSE=1 timeout 600 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C2_b.json 2> gpurun_out/bench_C2_b.err
IETI_VERBOSE=1 timeout 1200 python bench.py --config C5 --steps 3 --warmup 3 > gpurun_out/bench_C5_b.json 2> gpurun_out/bench_C5_b.err
timeout 600 python bench.py --config C5 --profile-iters 1 --no-e2e > gpurun_out/plain_C5.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_stencil \
  --launch-skip 2 -c 3 -o gpurun_out/sgs_C5_b python bench.py --config C5 --profile-iters 1 --no-e2e > gpurun_out/ncu_full_C5_b.log 2>&1
echo done
