#!/bin/bash
# pass aa: fused levels threshold (level 1 only vs levels 1-2), C3 tpr threshold A/B
mkdir -p gpurun_out
for FM in 24 100; do
  IETI_FUSE_MB=$FM timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5_aa_fm$FM.json 2> gpurun_out/bench_C5_aa_fm$FM.err
done
for TR in 40000 60000; do
  IETI_TPR1_ROWS=$TR timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C3_aa_tr$TR.json 2> gpurun_out/bench_C3_aa_tr$TR.err
done
echo done
