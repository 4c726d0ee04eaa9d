#!/bin/bash
# pass ac: concurrent problem groups on C5 level 2 (IETI_XG_SMALL) and finer x-groups (IETI_XGROUP_MB)
mkdir -p gpurun_out
for v in "a:" "b:IETI_XG_SMALL=2" "c:IETI_XG_SMALL=4" "d:IETI_XGROUP_MB=32" "e:IETI_XGROUP_MB=24" "f:IETI_XGROUP_MB=32 IETI_XG_SMALL=2"; do
  tag=${v%%:*}; envs=${v#*:}
  env $envs timeout 900 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_C5_${tag}_r2ac.json 2> /dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab_C5_${tag}_r2ac.json')); print('C5 [$envs]', round(d['value'],3), d['config']['pcg_iterations_per_solve'], round(d['ms_per_step'],1), 'frac', round(d['roofline']['frac'],3))"
done
