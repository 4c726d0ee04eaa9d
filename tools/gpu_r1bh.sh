#!/bin/bash
# pass bh: variant bench lines (NEXT-1 / NEXT-3) on the final build
mkdir -p gpurun_out
timeout 600 python bench.py --config C4 --local pcg --inner-tol 1e-12 --dirichlet pcg --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C4_dd_bh.json 2> gpurun_out/bench_C4_dd_bh.err
timeout 600 python bench.py --config C4 --local pcg --inner-tol 1e-12 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C4_mgd_bh.json 2> gpurun_out/bench_C4_mgd_bh.err
timeout 600 python bench.py --config C4 --local pcg --inner-tol 1e-10 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C4_mgmg_bh.json 2> gpurun_out/bench_C4_mgmg_bh.err
timeout 1200 python bench.py --config C5 --local pcg --inner-tol 1e-10 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5_mgmg_bh.json 2> gpurun_out/bench_C5_mgmg_bh.err
echo done
