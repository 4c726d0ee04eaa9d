#!/bin/bash
# pass al: interface kernels without block-wide reductions (warp per primal column, CSR of C rows, pool memset)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/pytest_gpu_r2al.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r2al.txt
tail -2 gpurun_out/pytest_gpu_r2al.txt
for v in "C4:" "C3:" "C2:" "C1:" "C5:"; do
  cfg=${v%%:*}; envs=${v#*:}
  st=10; [ $cfg = C5 ] && st=5
  env $envs timeout 900 python bench.py --config $cfg --steps $st --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_r2al.json 2> /dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab_r2al.json')); print('$cfg [$envs]', round(d['value'],3), d['config']['pcg_iterations_per_solve'], round(d['ms_per_step'],2), 'frac', round(d['roofline']['frac'],3))"
done
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_C4_r2al.csv python bench.py --config C4 --profile-iters 1 --no-cpu-baseline > /dev/null 2>&1
