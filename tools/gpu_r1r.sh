#!/bin/bash
# pass r: user-load test rework; full default bench (all keys) of C5; NEXT-1 (MG-MG) bench on C5 and C4
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r.log
timeout 1200 python bench.py > gpurun_out/bench_default_r.json 2> gpurun_out/bench_default_r.err
timeout 900 python bench.py --config C4 --local pcg --inner-tol 1e-10 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C4_mgmg_r.json 2> gpurun_out/bench_C4_mgmg_r.err
timeout 1500 python bench.py --config C5 --local pcg --inner-tol 1e-10 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5_mgmg_r.json 2> gpurun_out/bench_C5_mgmg_r.err
echo done
