#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_bf.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_bf.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_bf.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_bf.log
echo done
