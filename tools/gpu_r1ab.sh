#!/bin/bash
# pass ab: loopback two-rank test + full GPU suite
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k loopback > gpurun_out/pytest_gpu_ab_lb.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_ab_lb.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_ab.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_ab.log
echo done
