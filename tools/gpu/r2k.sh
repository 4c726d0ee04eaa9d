#!/bin/bash
# pass k: the whole GPU suite on the current build, smoke, and the default bench line
mkdir -p gpurun_out
export IETI_PARITY_LOG=$PWD/gpurun_out/parity_r2k.jsonl
rm -f $IETI_PARITY_LOG
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r2k.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r2k.txt
python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke_r2k.txt 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_r2k.txt
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_C5_r2k.json 2> gpurun_out/bench_C5_r2k.err
tail -3 gpurun_out/pytest_gpu_r2k.txt
