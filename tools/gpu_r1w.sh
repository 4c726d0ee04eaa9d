#!/bin/bash
# pass w: full GPU suite (NCCL 1-rank self-test, TMA variant), default bench, reference arm
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_w.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_w.log
IETI_VERBOSE=1 timeout 1200 python bench.py > gpurun_out/bench_default_w.json 2> gpurun_out/bench_default_w.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference_w.json 2> gpurun_out/bench_reference_w.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_w.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_w.log
echo done
