#!/bin/bash
mkdir -p gpurun_out
for k in 1 2 3; do timeout 300 python tools/determinism2.py C3 >> gpurun_out/det_az.log 2>&1; done
for k in 1 2; do timeout 300 python tools/determinism.py C3 >> gpurun_out/det_az.log 2>&1; done
timeout 900 python -m pytest tests -m gpu -q -x -k "C3s or C2s or loopback or nccl" > gpurun_out/pytest_gpu_az.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_az.log
echo done
