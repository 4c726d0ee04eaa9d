#!/bin/bash
# pass m: the whole GPU suite (nu_1 / nu_2, 2D p up to 7, direct solvers, MG-MG-S, full size), the
# default bench line, and Table 1's p = 7 shape (GS smoother: the paper's mass smoother is out of scope)
mkdir -p gpurun_out
export IETI_PARITY_LOG=$PWD/gpurun_out/parity_r2m.jsonl
rm -f $IETI_PARITY_LOG
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r2m.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r2m.txt
tail -3 gpurun_out/pytest_gpu_r2m.txt
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C5_r2m.json 2> gpurun_out/bench_C5_r2m.err
timeout 1200 python tools/paper_replica.py --p 7 --variant MGMG,DDX 32 64 > gpurun_out/replica_E1p7_r2m.jsonl 2>&1
cat gpurun_out/replica_E1p7_r2m.jsonl | cut -c1-220
