#!/bin/bash
# round-1 GPU pass: parity tests, bench C4/C5, ncu launch list + one full capture of the top kernel
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config C4 --steps 5 --warmup 3 > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err
timeout 1200 python bench.py --config C5 --steps 3 --warmup 3 > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches_C4.csv python bench.py --config C4 --profile-iters 1 > gpurun_out/ncu_list_C4.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_stencil \
  --launch-skip 0 -c 8 -o gpurun_out/sgs_C5 python bench.py --config C5 --profile-iters 1 --no-e2e > gpurun_out/ncu_full_C5.log 2>&1
echo done
