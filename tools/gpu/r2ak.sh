#!/bin/bash
# pass ak: C5 level 2 as a big (one thread per row, row-tiled) level with concurrent groups
mkdir -p gpurun_out
for v in "C5:" "C5:IETI_TPR1_ROWS=20000" "C5:IETI_TPR1_ROWS=20000 IETI_XG_BIG=2" "C5:IETI_TPR1_ROWS=20000 IETI_XG_BIG=4" "C5:IETI_XG_SMALL=4"; do
  cfg=${v%%:*}; envs=${v#*:}
  env $envs timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_r2ak.json 2> /dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab_r2ak.json')); print('$cfg [$envs]', round(d['value'],3), d['config']['pcg_iterations_per_solve'], round(d['ms_per_step'],2), 'frac', round(d['roofline']['frac'],3))"
done
