#!/bin/bash
# pass v: k_sweep_cl v5 (modes 6/7, global-coefficient mode)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cluster_sweep_bitwise" > gpurun_out/pytest_r2v.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_r2v.txt
tail -3 gpurun_out/pytest_r2v.txt
for cfg in C4 C3 C2 C1 C5; do
  for cl in 0 1; do
    IETI_VERBOSE=1 IETI_CLSWEEP=$cl timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${cfg}_cl${cl}_r2v.json 2> gpurun_out/ab_${cfg}_cl${cl}_r2v.err
    python -c "import json; d=json.load(open('gpurun_out/ab_${cfg}_cl${cl}_r2v.json')); print('$cfg cl$cl', round(d['value'],2), d['config']['pcg_iterations_per_solve'], round(d['ms_per_step'],3), 'frac', round(d['roofline']['frac'],3))" >> gpurun_out/ab_r2v_summary.txt 2>&1
  done
  grep -h "cluster sweep" gpurun_out/ab_${cfg}_cl1_r2v.err | head -4 >> gpurun_out/ab_r2v_summary.txt
done
cat gpurun_out/ab_r2v_summary.txt
for cfg in C4 C3; do
CMD="python bench.py --config $cfg --profile-iters 1"
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_${cfg}_cl_r2v.csv $CMD > /dev/null 2>&1
done
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_sweep_cl --launch-skip 4 --launch-count 4 -o gpurun_out/ncu_swcl_C3_r2v python bench.py --config C3 --profile-iters 1 > gpurun_out/ncu_swcl_r2v.log 2>&1
echo done
for cfg in C4 C3; do
  IETI_CLGLOBAL=1 timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${cfg}_clg_r2v.json 2> /dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab_${cfg}_clg_r2v.json')); print('$cfg clglobal', round(d['value'],2), d['config']['pcg_iterations_per_solve'], round(d['ms_per_step'],3))"
done
