#!/bin/bash
# A/B of the split-row finest-level kernel (k_stencil_split) and related switches on C5 / C3
mkdir -p gpurun_out
T=${TAG:-e}
run() {  # name, env..., then bench args after --
  local name=$1; shift
  local envs=()
  while [ "$1" != "--" ]; do envs+=("$1"); shift; done; shift
  env "${envs[@]}" timeout 900 python bench.py "$@" --no-cpu-baseline --no-e2e > gpurun_out/ab_${T}_${name}.json 2> gpurun_out/ab_${T}_${name}.err
  python -c "import json,sys; d=json.load(open('gpurun_out/ab_${T}_${name}.json')); r=d['roofline']; print('$name', round(d['value'],3), d['config']['pcg_iterations_per_solve'], 'frac', round(r['frac'],3), 'vcyc', {k: round(v,3) for k,v in r['all_levels_vcycles'].items() if isinstance(v,float)})" >> gpurun_out/ab_${T}_summary.txt 2>&1
}
run C5_base X=0 -- --config C5 --steps 2 --warmup 3
run C5_split1 IETI_SPLIT=1 -- --config C5 --steps 2 --warmup 3
run C5_split2 IETI_SPLIT=2 -- --config C5 --steps 2 --warmup 3
run C5_split2_l2big IETI_SPLIT=2 IETI_TPR1_ROWS=20000 -- --config C5 --steps 2 --warmup 3
run C5_split1_nogrp IETI_SPLIT=1 IETI_XGROUP_MB=0 -- --config C5 --steps 2 --warmup 3
run C5_split2_nogrp IETI_SPLIT=2 IETI_XGROUP_MB=0 -- --config C5 --steps 2 --warmup 3
run C3_base X=0 -- --config C3 --steps 5 --warmup 3
run C3_split2 IETI_SPLIT=2 -- --config C3 --steps 5 --warmup 3
cat gpurun_out/ab_${T}_summary.txt


