#!/bin/bash
# pass o: primal-basis chunk size A/B (C5 setup time), then bench lines of every config on this build
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "E1p7 or inner_pcg_cap" > gpurun_out/pytest_r2o.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_r2o.txt
mkdir -p gpurun_out
for mb in 32 128 256; do
  IETI_BASIS_MB=$mb timeout 900 python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/basis_mb${mb}_r2o.json 2> gpurun_out/basis_mb${mb}_r2o.err
  python -c "import json; d=json.load(open('gpurun_out/basis_mb${mb}_r2o.json')); print('basis_mb $mb', round(d['config']['setup_s'],1), d['config']['basis_pcg_iterations'], round(d['value'],3))" >> gpurun_out/basis_r2o_summary.txt
done
for cfg in C1 C2 C3 C4; do
  timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 > gpurun_out/bench_${cfg}_r2o.json 2> gpurun_out/bench_${cfg}_r2o.err
done
timeout 900 python bench.py --config C5 --steps 5 --warmup 3 > gpurun_out/bench_C5_r2o.json 2> gpurun_out/bench_C5_r2o.err
cat gpurun_out/basis_r2o_summary.txt
for cfg in C1 C2 C3 C4 C5; do python -c "import json; d=json.load(open('gpurun_out/bench_${cfg}_r2o.json')); print('$cfg', round(d['value'],2), d['config']['pcg_iterations_per_solve'], round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value'],2), 'setup', round(d['config']['setup_s'],1), 'frac', round(d['roofline']['frac'],3), 'cpu', d['cpu_baseline']['value'])"; done
