#!/bin/bash
# pass j: split rows with more (smaller) x-groups so that the phase's 2 threads per row stay one
# wave (64 registers: <= 151 k resident threads), wide k_full_t, TPR 8 on 2D p = 4
mkdir -p gpurun_out
T=j
run() {
  local name=$1; shift
  local envs=()
  while [ "$1" != "--" ]; do envs+=("$1"); shift; done; shift
  env "${envs[@]}" timeout 900 python bench.py "$@" --no-cpu-baseline --no-e2e > gpurun_out/ab_${T}_${name}.json 2> gpurun_out/ab_${T}_${name}.err
  python -c "import json,sys; d=json.load(open('gpurun_out/ab_${T}_${name}.json')); r=d['roofline']; print('$name', round(d['value'],3), d['config']['pcg_iterations_per_solve'], 'ms/it', round(d['config']['phases']['ms_per_iteration'],3), 'frac', round(r['frac'],3), 'vc', round(r['all_levels_vcycles']['algorithmic_gbs'],1))" >> gpurun_out/ab_${T}_summary.txt 2>&1
}
run C5 X=0 -- --config C5 --steps 2 --warmup 3
run C5_fullt0 IETI_FULLT=0 -- --config C5 --steps 2 --warmup 3
run C5_s1_xg32 IETI_SPLIT=1 IETI_XGROUP_MB=32 -- --config C5 --steps 2 --warmup 3
run C5_s1_xg24 IETI_SPLIT=1 IETI_XGROUP_MB=24 -- --config C5 --steps 2 --warmup 3
run C5_s1_xg19 IETI_SPLIT=1 IETI_XGROUP_MB=19 -- --config C5 --steps 2 --warmup 3
run C5_xg32 IETI_XGROUP_MB=32 -- --config C5 --steps 2 --warmup 3
run C3 X=0 -- --config C3 --steps 5 --warmup 3
run C3_s1 IETI_SPLIT=1 -- --config C3 --steps 5 --warmup 3
cat gpurun_out/ab_${T}_summary.txt
