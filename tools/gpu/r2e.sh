#!/bin/bash
# round 2 pass e: BPCG tests (s rounding), loopback whole-solve, split A/B, C3 basis-tolerance experiment
mkdir -p gpurun_out
export IETI_PARITY_LOG=$PWD/gpurun_out/parity_r2e.jsonl
rm -f $IETI_PARITY_LOG
timeout 900 python -m pytest tests/test_gpu_saddle.py -q > gpurun_out/pytest_saddle_r2e.txt 2>&1
echo "saddle rc=$?" >> gpurun_out/pytest_saddle_r2e.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "loopback or large_patches or edge_cases or zero_rhs" > gpurun_out/pytest_misc_r2e.txt 2>&1
echo "misc rc=$?" >> gpurun_out/pytest_misc_r2e.txt
timeout 900 python tools/gpu/c3_basis.py > gpurun_out/c3_basis_r2e.jsonl 2>&1
TAG=e bash tools/gpu/ab_split.sh
