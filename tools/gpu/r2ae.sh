#!/bin/bash
# pass ae: C5 launch list with DRAM bytes on the concurrent-group build (one fixed-iteration solve), C4/C3 lists
mkdir -p gpurun_out
CMD="python bench.py --config C5 --profile-iters 1 --no-cpu-baseline"
$CMD > gpurun_out/prof_plain_r2ae.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --profile-from-start off --csv --log-file gpurun_out/launches_C5_r2ae.csv $CMD > gpurun_out/ncu_r2ae.log 2>&1
echo "ncu rc=$?"
for cfg in C4 C3; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_${cfg}_r2ae.csv python bench.py --config $cfg --profile-iters 1 --no-cpu-baseline > /dev/null 2>&1
  echo "ncu $cfg rc=$?"
done
