#!/bin/bash
# pass ai: x replicated in shared memory per CTA (DSMEM broadcast of the updates): bitwise tests, A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cluster_sweep_bitwise" > gpurun_out/pytest_r2ai.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_r2ai.txt
tail -3 gpurun_out/pytest_r2ai.txt
for v in "C4:" "C4:IETI_CLREP=0" "C3:" "C3:IETI_CLREP=0" "C2:" "C2:IETI_CLREP=0" "C1:" "C5:"; do
  cfg=${v%%:*}; envs=${v#*:}
  st=10; [ $cfg = C5 ] && st=5
  env $envs IETI_VERBOSE=1 timeout 900 python bench.py --config $cfg --steps $st --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_r2ai.json 2> gpurun_out/ab_r2ai_${cfg}.err
  python -c "import json; d=json.load(open('gpurun_out/ab_r2ai.json')); print('$cfg [$envs]', round(d['value'],2), d['config']['pcg_iterations_per_solve'], round(d['ms_per_step'],3), 'frac', round(d['roofline']['frac'],3))"
done
grep -h "clusters resident" gpurun_out/ab_r2ai_C4.err | sort | uniq | head -12
