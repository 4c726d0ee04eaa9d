#!/bin/bash
# pass n: the new GPU tests, then the C5 launch list with DRAM bytes (one fixed-iteration solve)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "inner_pcg_cap or fixed_operator or smoothing_steps or edge_cases or direct or solve_parity or inner_pcg_counts" > gpurun_out/pytest_r2n.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_r2n.txt
tail -3 gpurun_out/pytest_r2n.txt
CMD="python bench.py --config C5 --profile-iters 1"
$CMD > gpurun_out/prof_plain_r2n.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --profile-from-start off --csv --log-file gpurun_out/launches_C5_r2n.csv $CMD > gpurun_out/ncu_r2n.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_r2n.log
tail -2 gpurun_out/ncu_r2n.log
