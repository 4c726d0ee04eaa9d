#!/bin/bash
# pass d: sum-factorised assembly + device-side basis PCG; parity, benches, C4 launch list, C5 ncu (warm L2)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_d.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_d.log
IETI_VERBOSE=1 timeout 600 python bench.py --config C4 --steps 5 --warmup 3 > gpurun_out/bench_C4_d.json 2> gpurun_out/bench_C4_d.err
IETI_VERBOSE=1 timeout 1200 python bench.py --config C5 --steps 3 --warmup 3 > gpurun_out/bench_C5_d.json 2> gpurun_out/bench_C5_d.err
timeout 300 python bench.py --config C4 --profile-iters 1 > gpurun_out/plain_C4.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches_C4_d.csv python bench.py --config C4 --profile-iters 1 > gpurun_out/ncu_list_C4_d.log 2>&1
timeout 400 python bench.py --config C5 --profile-iters 1 --no-e2e > gpurun_out/plain_C5_d.log 2>&1 && \
timeout 1500 ncu --set full --cache-control none --clock-control none --import-source on --profile-from-start off \
  -k regex:k_stencil --launch-skip 0 -c 6 -o gpurun_out/sgs_C5_d python bench.py --config C5 --profile-iters 1 --no-e2e > gpurun_out/ncu_full_C5_d.log 2>&1
echo done
