#!/bin/bash
# pass h: threads-per-row sensitivity of the latency-bound configs (C4, C3, the C5/8 per-rank proxy)
# and the ncu full capture of the finest (mode 7) / level-2 (mode 0) colour phases of C5
mkdir -p gpurun_out
T=h
run() {
  local name=$1; shift
  local envs=()
  while [ "$1" != "--" ]; do envs+=("$1"); shift; done; shift
  env "${envs[@]}" timeout 900 python bench.py "$@" --no-cpu-baseline --no-e2e > gpurun_out/ab_${T}_${name}.json 2> gpurun_out/ab_${T}_${name}.err
  python -c "import json,sys; d=json.load(open('gpurun_out/ab_${T}_${name}.json')); r=d['roofline']; print('$name', round(d['value'],3), d['config']['pcg_iterations_per_solve'], 'ms/it', round(d['config']['phases']['ms_per_iteration'],3))" >> gpurun_out/ab_${T}_summary.txt 2>&1
}
for t in 4 8 16; do run C4_tpr$t IETI_TPR=$t -- --config C4 --steps 10 --warmup 3; done
for t in 4 8 16; do run C3_tpr$t IETI_TPR=$t -- --config C3 --steps 5 --warmup 3; done
run C3_big1 IETI_TPR1_ROWS=1000000 -- --config C3 --steps 5 --warmup 3
for t in 4 8 16; do run C5g442_tpr$t IETI_TPR=$t -- --config C5 --grid 4,4,2 --steps 3 --warmup 3; done
run C5g442_nopdl IETI_PDL=0 -- --config C5 --grid 4,4,2 --steps 3 --warmup 3
run C5g442_fuse IETI_FUSE=1 -- --config C5 --grid 4,4,2 --steps 3 --warmup 3
cat gpurun_out/ab_${T}_summary.txt
CMD="python bench.py --config C5 --profile-iters 1"
$CMD > gpurun_out/prof_plain_r2h.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:k_stencil<.int.3, .int.3, .int.(1, .int.7|8, .int.0),' -c 4 --profile-from-start off \
    -o gpurun_out/prof_sgs_r2h $CMD > gpurun_out/ncu_r2h.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_r2h.log
tail -3 gpurun_out/ncu_r2h.log
