#!/bin/bash
# Build here (nvcc cross-compile) and only then ship the repo + run <script> on a B200 via gpurun.
# usage: tools/gpu_submit.sh <script> [timeout_s]   (output: /tmp/gpurun_<name>.log)
set -e
cd "$(dirname "$0")/.."
python -c 'import __graft_entry__ as g; g.build()'
name=$(basename "$1" .sh)
/usr/local/graft/bin/gpurun --timeout "${2:-3000}" -- "bash $1" > /tmp/gpurun_${name}.log 2>&1
