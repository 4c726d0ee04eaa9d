#!/bin/bash
# pass q: cluster sweep (k_sweep_cl) bitwise test, then A/B C4 / C3 / C2 / C1 with IETI_CLSWEEP=0/1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cluster_sweep_bitwise" > gpurun_out/pytest_r2q.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_r2q.txt
tail -3 gpurun_out/pytest_r2q.txt
for cfg in C4 C3 C2 C1; do
  for cl in 0 1; do
    IETI_VERBOSE=1 IETI_CLSWEEP=$cl timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${cfg}_cl${cl}_r2q.json 2> gpurun_out/ab_${cfg}_cl${cl}_r2q.err
    python -c "import json; d=json.load(open('gpurun_out/ab_${cfg}_cl${cl}_r2q.json')); print('$cfg cl$cl', round(d['value'],2), d['config']['pcg_iterations_per_solve'], round(d['ms_per_step'],3), 'frac', round(d['roofline']['frac'],3))" >> gpurun_out/ab_r2q_summary.txt 2>&1
  done
done
cat gpurun_out/ab_r2q_summary.txt
grep -h "cluster sweep" gpurun_out/ab_*_cl1_r2q.err | sort | uniq | head -20
