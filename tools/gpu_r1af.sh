#!/bin/bash
# pass af: level 2 as a big level (offset-major, 1 thread per row) A/B
mkdir -p gpurun_out
for TR in 40000 20000; do
  IETI_TPR1_ROWS=$TR timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5_af_tr$TR.json 2> gpurun_out/bench_C5_af_tr$TR.err
done
echo done
