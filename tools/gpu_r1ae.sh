#!/bin/bash
# pass ae: 2 threads per row on the big levels (A/B); paper replica with 4x8 orientation; parity of big path
mkdir -p gpurun_out
for TB in 1 2; do
  IETI_TPR_BIG=$TB timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5_ae_tb$TB.json 2> gpurun_out/bench_C5_ae_tb$TB.err
done
IETI_TPR_BIG=2 timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C3_ae_tb2.json 2> gpurun_out/bench_C3_ae_tb2.err
timeout 1500 python tools/paper_replica.py --grid 4,8 64 128 256 512 > gpurun_out/paper_replica_ae_4x8.jsonl 2> gpurun_out/paper_replica_ae.err
IETI_TPR_BIG=2 IETI_TPR=1 timeout 900 python -m pytest tests -m gpu -q -k "large" > gpurun_out/pytest_gpu_ae.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_ae.log
echo done
