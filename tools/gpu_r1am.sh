#!/bin/bash
# pass am: unrolled transfer kernels; full suite, all configs, C5 launch list
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_am.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_am.log
for C in C4 C3 C2 C1; do
  timeout 600 python bench.py --config $C --steps 5 --warmup 3 > gpurun_out/bench_${C}_am.json 2> gpurun_out/bench_${C}_am.err
done
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5_am.json 2> gpurun_out/bench_C5_am.err
timeout 400 python bench.py --config C5 --profile-iters 1 --no-e2e > gpurun_out/plain_C5_am.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches_C5_am.csv python bench.py --config C5 --profile-iters 1 --no-e2e > gpurun_out/ncu_list_C5_am.log 2>&1
echo done
