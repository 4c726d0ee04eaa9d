#!/bin/bash
# pass ag: C5 level 1 through cluster sweeps instead of the fused V-cycle kernel (IETI_FUSE=0)
mkdir -p gpurun_out
for v in "C5:IETI_FUSE=0" "C5:" ; do
  cfg=${v%%:*}; envs=${v#*:}
  env $envs IETI_VERBOSE=1 timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_r2ag.json 2> gpurun_out/ab_r2ag.err
  python -c "import json; d=json.load(open('gpurun_out/ab_r2ag.json')); print('$cfg [$envs]', round(d['value'],3), d['config']['pcg_iterations_per_solve'], round(d['ms_per_step'],1), 'frac', round(d['roofline']['frac'],3))"
  grep "of 256 clusters" gpurun_out/ab_r2ag.err | head -4
done
