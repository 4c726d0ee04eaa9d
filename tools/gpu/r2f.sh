#!/bin/bash
# pass f: persistent sweep (IETI_PSWEEP) parity and A/B on C5 / C4 / C3 / C2
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "persistent_sweep" > gpurun_out/pytest_psweep_r2f.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_psweep_r2f.txt
tail -3 gpurun_out/pytest_psweep_r2f.txt
T=f
run() {
  local name=$1; shift
  local envs=()
  while [ "$1" != "--" ]; do envs+=("$1"); shift; done; shift
  env "${envs[@]}" timeout 900 python bench.py "$@" --no-cpu-baseline --no-e2e > gpurun_out/ab_${T}_${name}.json 2> gpurun_out/ab_${T}_${name}.err
  python -c "import json,sys; d=json.load(open('gpurun_out/ab_${T}_${name}.json')); r=d['roofline']; print('$name', round(d['value'],3), d['config']['pcg_iterations_per_solve'], 'frac', round(r['frac'],3), 'vcyc_alg', round(r['all_levels_vcycles']['algorithmic_gbs'],1), 'ms/it', round(d['config']['phases']['ms_per_iteration'],3))" >> gpurun_out/ab_${T}_summary.txt 2>&1
}
run C5_base X=0 -- --config C5 --steps 2 --warmup 3
run C5_psweep IETI_PSWEEP=1 -- --config C5 --steps 2 --warmup 3
run C4_base X=0 -- --config C4 --steps 10 --warmup 3
run C4_psweep IETI_PSWEEP=1 -- --config C4 --steps 10 --warmup 3
run C3_base X=0 -- --config C3 --steps 5 --warmup 3
run C3_psweep IETI_PSWEEP=1 -- --config C3 --steps 5 --warmup 3
run C2_base X=0 -- --config C2 --steps 10 --warmup 3
run C2_psweep IETI_PSWEEP=1 -- --config C2 --steps 10 --warmup 3
run C5_psweep_nofuse IETI_PSWEEP=1 IETI_FUSE=0 -- --config C5 --steps 2 --warmup 3
cat gpurun_out/ab_${T}_summary.txt
