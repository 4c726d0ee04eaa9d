#!/bin/bash
# pass ad: 16-deep load batches on the finest level (A/B); paper replica E1 (MG-MG, m = 64..512)
mkdir -p gpurun_out
for NB in 8 16; do
  IETI_BATCH=$NB timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5_ad_nb$NB.json 2> gpurun_out/bench_C5_ad_nb$NB.err
done
timeout 1500 python tools/paper_replica.py 64 128 256 512 > gpurun_out/paper_replica_ad.jsonl 2> gpurun_out/paper_replica_ad.err
echo done
