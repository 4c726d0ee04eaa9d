#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "full_size" --durations=3 > gpurun_out/pytest_gpu_ap.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_ap.log
echo done
