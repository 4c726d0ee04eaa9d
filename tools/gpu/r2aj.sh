#!/bin/bash
# pass aj: row-tiled coefficients on the big levels (IETI_TILE): GPU suite, A/B C5 / C3
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/pytest_gpu_r2aj.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r2aj.txt
tail -2 gpurun_out/pytest_gpu_r2aj.txt
for v in "C5:" "C5:IETI_TILE=0" "C3:" "C3:IETI_TILE=0"; do
  cfg=${v%%:*}; envs=${v#*:}
  st=10; [ $cfg = C5 ] && st=5
  env $envs timeout 900 python bench.py --config $cfg --steps $st --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_r2aj.json 2> /dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab_r2aj.json')); print('$cfg [$envs]', round(d['value'],3), d['config']['pcg_iterations_per_solve'], round(d['ms_per_step'],2), 'frac', round(d['roofline']['frac'],3))"
done
