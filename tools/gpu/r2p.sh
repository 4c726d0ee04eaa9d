#!/bin/bash
# pass p: basis chunk sizes 1024 / 4096 MB with the setup-stage breakdown, then the whole GPU suite
mkdir -p gpurun_out
for mb in 256 1024 4096; do
  IETI_VERBOSE=1 IETI_BASIS_MB=$mb timeout 900 python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/basis_mb${mb}_r2p.json 2> gpurun_out/basis_mb${mb}_r2p.err
  python -c "import json; d=json.load(open('gpurun_out/basis_mb${mb}_r2p.json')); print('basis_mb $mb', round(d['config']['setup_s'],1), d['config']['basis_pcg_iterations'], round(d['value'],3))" >> gpurun_out/basis_r2p_summary.txt
done
cat gpurun_out/basis_r2p_summary.txt
export IETI_PARITY_LOG=$PWD/gpurun_out/parity_r2p.jsonl
rm -f $IETI_PARITY_LOG
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r2p.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r2p.txt
tail -3 gpurun_out/pytest_gpu_r2p.txt
