#!/bin/bash
# pass ac: ncu --set full of the finest MODE-0 half-phase (x-resident groups), warm L2
mkdir -p gpurun_out
timeout 400 python bench.py --config C5 --profile-iters 1 --no-e2e > gpurun_out/plain_C5_ac.log 2>&1 && \
timeout 1500 ncu --set full --cache-control none --clock-control none --import-source on --profile-from-start off \
  --kernel-name-base demangled -k "regex:k_stencil<.int.3, .int.3, .int.1, .int.0>" --launch-skip 128 -c 3 -o gpurun_out/sgs_C5_ac \
  python bench.py --config C5 --profile-iters 1 --no-e2e > gpurun_out/ncu_full_C5_ac.log 2>&1
echo done
