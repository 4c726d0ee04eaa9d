#!/bin/bash
# Host facts of the GPU box (cores, RAM, CPU model) + the GPU suite on the current build.
mkdir -p gpurun_out
{ nproc; lscpu | head -30; free -g; nvidia-smi -L; python -c 'import os; print("cpu_count", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))'; } > gpurun_out/host_r2.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r2a.txt 2>&1
echo rc=$?
