#!/bin/bash
# pass an: ncu --set full of the finest prolongation and restriction
mkdir -p gpurun_out
timeout 400 python bench.py --config C5 --profile-iters 1 --no-e2e > gpurun_out/plain_C5_an.log 2>&1
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on --profile-from-start off \
  --kernel-name-base demangled -k "regex:k_prolong" --launch-skip 1 -c 1 -o gpurun_out/prolong_C5_an \
  python bench.py --config C5 --profile-iters 1 --no-e2e > gpurun_out/ncu_prolong_an.log 2>&1
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on --profile-from-start off \
  --kernel-name-base demangled -k "regex:k_restrict" -c 1 -o gpurun_out/restrict_C5_an \
  python bench.py --config C5 --profile-iters 1 --no-e2e > gpurun_out/ncu_restrict_an.log 2>&1
echo done
