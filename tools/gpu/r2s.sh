#!/bin/bash
# pass s: where does a k_sweep_cl phase spend its time (C3: cluster sweeps on levels 1-4)
mkdir -p gpurun_out
CMD="python bench.py --config C3 --profile-iters 1"
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_C3_cl_r2s.csv $CMD > /dev/null 2>&1
IETI_CLSWEEP=0 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_C3_nocl_r2s.csv $CMD > /dev/null 2>&1
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_sweep_cl --launch-skip 4 --launch-count 4 -o gpurun_out/ncu_swcl_C3_r2s $CMD > gpurun_out/ncu_swcl_r2s.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_swcl_r2s.log
