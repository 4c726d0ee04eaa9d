#!/bin/bash
# pass z: fixed dynamic-smem ceiling per k_sweep_cl instance (ncu replays), bitwise test, A/B, launch lists
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cluster_sweep_bitwise" > gpurun_out/pytest_r2z.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_r2z.txt
tail -2 gpurun_out/pytest_r2z.txt
for cfg in C4 C3 C2 C1; do
  timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${cfg}_r2z.json 2> /dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab_${cfg}_r2z.json')); print('$cfg', round(d['value'],2), d['config']['pcg_iterations_per_solve'], round(d['ms_per_step'],3), 'phase_us', round(d['roofline']['avg_launch_us'],2))"
done
for cfg in C4 C3 C2; do
  ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_${cfg}_r2z.csv python bench.py --config $cfg --profile-iters 1 --no-cpu-baseline > gpurun_out/ncu_${cfg}_r2z.log 2>&1
  echo "ncu $cfg rc=$?"
done
