#!/bin/bash
# pass t: C5 launch list (time + DRAM bytes per launch) and ncu --set full of finest MODE-0 phases
mkdir -p gpurun_out
timeout 400 python bench.py --config C5 --profile-iters 1 --no-e2e > gpurun_out/plain_C5_t.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches_C5_t.csv python bench.py --config C5 --profile-iters 1 --no-e2e > gpurun_out/ncu_list_C5_t.log 2>&1
timeout 1500 ncu --set full --cache-control none --clock-control none --import-source on --profile-from-start off \
  --kernel-name-base demangled -k regex:"k_stencil<3, 3, 1, 0>" --launch-skip 64 -c 3 -o gpurun_out/sgs_C5_t \
  python bench.py --config C5 --profile-iters 1 --no-e2e > gpurun_out/ncu_full_C5_t.log 2>&1
echo done
