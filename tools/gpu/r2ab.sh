#!/bin/bash
# pass ab: x-groups of a finest-level sweep on concurrent graph branches (C5)
mkdir -p gpurun_out
for xc in 0 1 0 1; do
  IETI_XGCONC=$xc timeout 900 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_C5_xg${xc}_r2ab.json 2> /dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab_C5_xg${xc}_r2ab.json')); print('C5 xgconc $xc', round(d['value'],3), d['config']['pcg_iterations_per_solve'], round(d['ms_per_step'],1), 'phase_us', round(d['roofline']['avg_launch_us'],2), 'frac', round(d['roofline']['frac'],3))"
done
timeout 1500 python -m pytest tests/test_gpu_full_size.py -q -x -k "C5" > gpurun_out/pytest_full_r2ab.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_full_r2ab.txt; tail -2 gpurun_out/pytest_full_r2ab.txt
