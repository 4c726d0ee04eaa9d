#!/bin/bash
# pass g: BPCG tests (lambda scale), per-rank proxies of C5 at 2/4/8 GPUs, ncu full capture of the
# finest-level (mode 7) and level-2 (mode 0) colour-phase kernels
mkdir -p gpurun_out
export IETI_PARITY_LOG=$PWD/gpurun_out/parity_r2g.jsonl
rm -f $IETI_PARITY_LOG
timeout 900 python -m pytest tests/test_gpu_saddle.py -q > gpurun_out/pytest_saddle_r2g.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_saddle_r2g.txt
for g in 4,8,4 4,4,4 4,4,2; do
  timeout 900 python bench.py --config C5 --grid $g --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/proxy_C5_${g//,/x}.json 2> gpurun_out/proxy_C5_${g//,/x}.err
done
CMD="python bench.py --config C5 --profile-iters 1"
$CMD > gpurun_out/prof_plain_r2g.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:k_stencil<3, 3, (1, 7|8, 0),' -c 4 --profile-from-start off \
    -o gpurun_out/prof_sgs_r2g $CMD > gpurun_out/ncu_r2g.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_r2g.log
tail -3 gpurun_out/ncu_r2g.log
