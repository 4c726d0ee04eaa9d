#!/bin/bash
# pass aa: k_coarse row splits; C3 finest level as a row-major (cluster-swept) level
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cluster_sweep_bitwise or vcycle_and_local or solve_parity" > gpurun_out/pytest_r2aa.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_r2aa.txt
tail -2 gpurun_out/pytest_r2aa.txt
for v in "C4:" "C3:" "C2:" "C1:" "C3:IETI_TPR1_ROWS=100000" "C3:IETI_TPR1_ROWS=100000 IETI_CLMAX_MB=0" "C5:"; do
  cfg=${v%%:*}; envs=${v#*:}
  st=10; [ $cfg = C5 ] && st=5
  env $envs timeout 900 python bench.py --config $cfg --steps $st --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_r2aa.json 2> /dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab_r2aa.json')); print('$cfg [$envs]', round(d['value'],2), d['config']['pcg_iterations_per_solve'], round(d['ms_per_step'],3), 'phase_us', round(d['roofline']['avg_launch_us'],2), 'frac', round(d['roofline']['frac'],3))"
done
