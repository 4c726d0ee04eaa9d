#!/bin/bash
# pass q: diag/b loads off the critical path; NEXT-1 + user-load tests
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_q.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_q.log
for C in C4 C2 C3 C1; do
  timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${C}_q.json 2> gpurun_out/bench_${C}_q.err
done
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5_q.json 2> gpurun_out/bench_C5_q.err
echo done
