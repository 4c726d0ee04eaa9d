#!/bin/bash
# pass ah: full GPU suite + bench lines (C5 level 1 cluster-swept instead of fused)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_gpu_r2ah.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r2ah.txt
tail -3 gpurun_out/pytest_gpu_r2ah.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2ah.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_r2ah.txt
tail -2 gpurun_out/smoke_r2ah.txt
for cfg in C1 C2 C3 C4; do
  timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 > gpurun_out/bench_${cfg}_r2ah.json 2> gpurun_out/bench_${cfg}_r2ah.err
done
timeout 900 python bench.py --config C5 --steps 5 --warmup 3 > gpurun_out/bench_C5_r2ah.json 2> gpurun_out/bench_C5_r2ah.err
for cfg in C1 C2 C3 C4 C5; do python -c "import json; d=json.load(open('gpurun_out/bench_${cfg}_r2ah.json')); print('$cfg', round(d['value'],2), d['config']['pcg_iterations_per_solve'], round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value'],2), 'setup', round(d['config']['setup_s'],1), 'frac', round(d['roofline']['frac'],3), 'gpu_launches', d.get('gpu_launches'), 'cpu', d['cpu_baseline']['value'])"; done
