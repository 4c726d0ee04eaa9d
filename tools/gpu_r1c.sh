#!/bin/bash
# pass c: parity after the half-stream V-cycle modes (MODE 4/5) + C5/C4 bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_c.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_c.log
timeout 600 python bench.py --config C4 --steps 5 --warmup 3 > gpurun_out/bench_C4_c.json 2> gpurun_out/bench_C4_c.err
IETI_VERBOSE=1 timeout 1200 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C5_c.json 2> gpurun_out/bench_C5_c.err
echo done
