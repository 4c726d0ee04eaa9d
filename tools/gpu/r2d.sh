#!/bin/bash
# round 2 pass d: MG-MG-S (BPCG) tests, full GPU suite (full-size C2-C5), bench lines, paper replicas,
# and the whole-solve oracle timings on the host cores (background, after the bench lines)
mkdir -p gpurun_out
export IETI_PARITY_LOG=$PWD/gpurun_out/parity_r2d.jsonl
rm -f $IETI_PARITY_LOG
timeout 900 python -m pytest tests/test_gpu_saddle.py -x -q > gpurun_out/pytest_saddle_r2d.txt 2>&1
echo "saddle rc=$?" >> gpurun_out/pytest_saddle_r2d.txt
timeout 600 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C5_r2d.json 2> gpurun_out/bench_C5_r2d.err
timeout 900 python bench.py --config C5 --outer bpcg --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5_bpcg_r2d.json 2> gpurun_out/bench_C5_bpcg_r2d.err
timeout 600 python bench.py --config C4 --outer bpcg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C4_bpcg_r2d.json 2> gpurun_out/bench_C4_bpcg_r2d.err
export OMP_NUM_THREADS=1
nohup timeout 2400 python tools/oracle_full_runs.py C1 C2 C4 C3 --workers 8 --out gpurun_out/oracle_full_runs.json > gpurun_out/oracle_full_runs.log 2>&1 &
OPID=$!
timeout 900 python tools/paper_replica.py --variant MGMGS 64 128 256 > gpurun_out/replica_E1_mgmgs_r2d.jsonl 2>&1
timeout 900 python tools/paper_replica.py --workload E2 --variant MGMGS 4 8 16 > gpurun_out/replica_E2_mgmgs_r2d.jsonl 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r2d.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r2d.txt
wait $OPID
tail -3 gpurun_out/pytest_gpu_r2d.txt
