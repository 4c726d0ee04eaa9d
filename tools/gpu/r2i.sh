#!/bin/bash
# pass i: 9 blocks/SM for the multi-thread-per-row stencil levels (one wave for C5's level-2
# phases) on C5 / C4 / C3 / C2 / the C5/8 proxy; ncu full capture of C5's finest mode-7 phases
mkdir -p gpurun_out
T=i
run() {
  local name=$1; shift
  local envs=()
  while [ "$1" != "--" ]; do envs+=("$1"); shift; done; shift
  env "${envs[@]}" timeout 900 python bench.py "$@" --no-cpu-baseline --no-e2e > gpurun_out/ab_${T}_${name}.json 2> gpurun_out/ab_${T}_${name}.err
  python -c "import json,sys; d=json.load(open('gpurun_out/ab_${T}_${name}.json')); r=d['roofline']; print('$name', round(d['value'],3), d['config']['pcg_iterations_per_solve'], 'ms/it', round(d['config']['phases']['ms_per_iteration'],3), 'frac', round(r['frac'],3))" >> gpurun_out/ab_${T}_summary.txt 2>&1
}
run C5 X=0 -- --config C5 --steps 2 --warmup 3
run C4 X=0 -- --config C4 --steps 10 --warmup 3
run C3 X=0 -- --config C3 --steps 5 --warmup 3
run C3_tpr8 IETI_TPR=8 -- --config C3 --steps 5 --warmup 3
run C2 X=0 -- --config C2 --steps 10 --warmup 3
run C2_tpr8 IETI_TPR=8 -- --config C2 --steps 10 --warmup 3
run C5g442 X=0 -- --config C5 --grid 4,4,2 --steps 3 --warmup 3
cat gpurun_out/ab_${T}_summary.txt
CMD="python bench.py --config C5 --profile-iters 1"
$CMD > gpurun_out/prof_plain_r2i.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:k_stencil<.int.3, .int.3, .int.1, .int.7' -c 2 --profile-from-start off \
    -o gpurun_out/prof_sgs7_r2i $CMD > gpurun_out/ncu_r2i.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_r2i.log
