#!/bin/bash
# pass r: k_sweep_cl v2 (row state + all gathers issued before / right after the barrier): bitwise test, A/B, ncu
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cluster_sweep_bitwise" > gpurun_out/pytest_r2r.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_r2r.txt
tail -3 gpurun_out/pytest_r2r.txt
for cfg in C4 C3 C2 C1; do
  for cl in 0 1; do
    IETI_CLSWEEP=$cl timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${cfg}_cl${cl}_r2r.json 2> gpurun_out/ab_${cfg}_cl${cl}_r2r.err
    python -c "import json; d=json.load(open('gpurun_out/ab_${cfg}_cl${cl}_r2r.json')); print('$cfg cl$cl', round(d['value'],2), d['config']['pcg_iterations_per_solve'], round(d['ms_per_step'],3), 'frac', round(d['roofline']['frac'],3))" >> gpurun_out/ab_r2r_summary.txt 2>&1
  done
done
cat gpurun_out/ab_r2r_summary.txt
CMD="python bench.py --config C4 --profile-iters 1"
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_sweep_cl --launch-skip 8 --launch-count 3 -o gpurun_out/ncu_swcl_C4_r2r $CMD > gpurun_out/ncu_swcl_r2r.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_swcl_r2r.log
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_C4_cl_r2r.csv $CMD > /dev/null 2>&1
IETI_CLSWEEP=0 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_C4_nocl_r2r.csv $CMD > /dev/null 2>&1
echo done
