#!/bin/bash
# pass ai: fault injection + NEXT-3 exact variants, then full suite
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "fault or next3 or next1" > gpurun_out/pytest_gpu_ai1.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_ai1.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_ai.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_ai.log
echo done
