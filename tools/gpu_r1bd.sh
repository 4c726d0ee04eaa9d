#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "cycle_boundary" > gpurun_out/pytest_gpu_bd.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_bd.log
echo done
