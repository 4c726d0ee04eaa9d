#!/bin/bash
# pass h: offset tables in global memory, tpr 1/4/8 per level, fusion opt-in
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_h.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_h.log
IETI_VERBOSE=1 timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5_h.json 2> gpurun_out/bench_C5_h.err
for C in C4 C3 C2 C1; do
  timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${C}_h.json 2> gpurun_out/bench_${C}_h.err
done
timeout 300 python bench.py --config C4 --profile-iters 1 > gpurun_out/plain_C4_h.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches_C4_h.csv python bench.py --config C4 --profile-iters 1 > gpurun_out/ncu_list_C4_h.log 2>&1
echo done
