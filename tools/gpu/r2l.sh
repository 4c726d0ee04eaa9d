#!/bin/bash
# pass l: direct local solvers (batched banded Cholesky: D-D / MG-D as the paper scopes them), full-size
# parity re-run, replicas of Table 1 / 2 with the direct variants
mkdir -p gpurun_out
export IETI_PARITY_LOG=$PWD/gpurun_out/parity_r2l.jsonl
rm -f $IETI_PARITY_LOG
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_size.py -q -k "direct or full_size" > gpurun_out/pytest_direct_r2l.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_direct_r2l.txt
tail -3 gpurun_out/pytest_direct_r2l.txt
timeout 1200 python tools/paper_replica.py --variant DDX,MGDX,DD 64 128 256 > gpurun_out/replica_E1_direct_r2l.jsonl 2>&1
timeout 1200 python tools/paper_replica.py --workload E2 --variant DDX,MGDX 4 8 16 32 > gpurun_out/replica_E2_direct_r2l.jsonl 2>&1
timeout 900 python bench.py --config C4 --local direct --dirichlet direct --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C4_ddx_r2l.json 2> gpurun_out/bench_C4_ddx_r2l.err
cat gpurun_out/replica_E1_direct_r2l.jsonl gpurun_out/replica_E2_direct_r2l.jsonl | cut -c1-200
