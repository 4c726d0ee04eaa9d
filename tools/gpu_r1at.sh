#!/bin/bash
# pass at: ncu --set full of the finest MODE-0 phase (final code); largest paper rows (E1 m=1024, E2 m=32) MG-MG
mkdir -p gpurun_out
timeout 400 python bench.py --config C5 --profile-iters 1 --no-e2e > gpurun_out/plain_C5_at.log 2>&1
timeout 1500 ncu --set full --cache-control none --clock-control none --import-source on --profile-from-start off \
  --kernel-name-base demangled -k "regex:k_stencil<.int.3, .int.3, .int.1, .int.0" --launch-skip 64 -c 2 -o gpurun_out/sgs_C5_at \
  python bench.py --config C5 --profile-iters 1 --no-e2e > gpurun_out/ncu_full_C5_at.log 2>&1
timeout 1200 python tools/paper_replica.py --workload E1 --grid 4,8 --variant MGMG,MGD 1024 > gpurun_out/replica_E1_1024.jsonl 2> gpurun_out/replica_E1_1024.err
timeout 1200 python tools/paper_replica.py --workload E2 --grid 4,8,4 --variant MGMG,MGD 32 > gpurun_out/replica_E2_32.jsonl 2> gpurun_out/replica_E2_32.err
echo done
