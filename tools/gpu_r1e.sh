#!/bin/bash
# pass e: primal basis by PCG on K (+ bordered floating systems), cp.async-pipelined fine stencil kernel
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_e.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_e.log
IETI_VERBOSE=1 timeout 1200 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C5_e.json 2> gpurun_out/bench_C5_e.err
IETI_VERBOSE=1 timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C4_e.json 2> gpurun_out/bench_C4_e.err
timeout 400 python bench.py --config C5 --profile-iters 1 --no-e2e > gpurun_out/plain_C5_e.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches_C5_e.csv python bench.py --config C5 --profile-iters 1 --no-e2e > gpurun_out/ncu_list_C5_e.log 2>&1
echo done
