#!/bin/bash
# pass x: k_sweep_cl with batched coefficient+gather loads in global-coefficient mode
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cluster_sweep_bitwise" > gpurun_out/pytest_r2x.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_r2x.txt
tail -3 gpurun_out/pytest_r2x.txt
for cfg in C4 C3 C2; do
  for v in "cl1:IETI_CLSWEEP=1" "clg:IETI_CLGLOBAL=1"; do
    tag=${v%%:*}; envs=${v#*:}
    env $envs timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${cfg}_${tag}_r2x.json 2> gpurun_out/ab_${cfg}_${tag}_r2x.err
    python -c "import json; d=json.load(open('gpurun_out/ab_${cfg}_${tag}_r2x.json')); print('$cfg $tag', round(d['value'],2), d['config']['pcg_iterations_per_solve'], round(d['ms_per_step'],3), 'phase_us', round(d['roofline']['avg_launch_us'],2))"
  done
done
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_C4_cl_r2x.csv python bench.py --config C4 --profile-iters 1 > gpurun_out/ncu_C4_r2x.log 2>&1
echo "ncu rc=$?"; grep -i "error\|warn" gpurun_out/ncu_C4_r2x.log | head -5
