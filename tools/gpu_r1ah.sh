#!/bin/bash
# pass ah: full GPU suite (fault injection), smoke
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_ah.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_ah.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_ah.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_ah.log
echo done
