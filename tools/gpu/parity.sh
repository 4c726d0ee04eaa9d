#!/bin/bash
# GPU parity suite with the realized errors logged (profiles/r02/parity_*.jsonl after copying).
# usage: bash tools/gpu/parity.sh <tag> [pytest -k expression]
mkdir -p gpurun_out
tag=${1:-x}
export IETI_PARITY_LOG=$PWD/gpurun_out/parity_$tag.jsonl
rm -f "$IETI_PARITY_LOG"
if [ -n "$2" ]; then
  timeout 2400 python -m pytest tests -m gpu -q -k "$2" > gpurun_out/pytest_gpu_$tag.txt 2>&1
else
  timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$tag.txt 2>&1
fi
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$tag.txt
tail -3 gpurun_out/pytest_gpu_$tag.txt
