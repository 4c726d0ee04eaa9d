#!/bin/bash
# pass f: TMA-fed fine-level stencil kernel, L2-sized basis chunks
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_f.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_f.log
IETI_VERBOSE=1 timeout 1200 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C5_f.json 2> gpurun_out/bench_C5_f.err
IETI_VERBOSE=1 timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C3_f.json 2> gpurun_out/bench_C3_f.err
timeout 400 python bench.py --config C5 --profile-iters 1 --no-e2e > gpurun_out/plain_C5_f.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches_C5_f.csv python bench.py --config C5 --profile-iters 1 --no-e2e > gpurun_out/ncu_list_C5_f.log 2>&1
echo done
