#!/bin/bash
# pass y: why does ncu stop at the first k_sweep_cl mode-0 launch (C4)?
mkdir -p gpurun_out
CMD="python bench.py --config C4 --profile-iters 1 --no-cpu-baseline"
$CMD > gpurun_out/y0.log 2>&1; echo "plain rc=$?"; tail -2 gpurun_out/y0.log
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off $CMD > gpurun_out/y1.log 2>&1; echo "ncu rc=$?"; grep -v "^  \|^    " gpurun_out/y1.log | tail -12
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --replay-mode application $CMD > gpurun_out/y2.log 2>&1; echo "ncu app-replay rc=$?"; grep -c "k_sweep_cl" gpurun_out/y2.log; tail -3 gpurun_out/y2.log
IETI_CLGLOBAL=1 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off $CMD > gpurun_out/y3.log 2>&1; echo "ncu clglobal rc=$?"; grep -c "k_sweep_cl" gpurun_out/y3.log; tail -3 gpurun_out/y3.log
