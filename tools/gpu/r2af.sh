#!/bin/bash
# pass af: at least 2 concurrent groups on the big levels (C3's finest level), A/B
mkdir -p gpurun_out
for v in "C3:" "C3:IETI_XG_BIG=2" "C3:IETI_XG_BIG=4" "C4:" "C4:IETI_XG_BIG=2" "C5:IETI_XG_BIG=4"; do
  cfg=${v%%:*}; envs=${v#*:}
  st=10; [ $cfg = C5 ] && st=5
  env $envs timeout 900 python bench.py --config $cfg --steps $st --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_r2af.json 2> /dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab_r2af.json')); print('$cfg [$envs]', round(d['value'],2), d['config']['pcg_iterations_per_solve'], round(d['ms_per_step'],3), 'frac', round(d['roofline']['frac'],3))"
done
