#!/bin/bash
# pass au: modes 6/7 (backward sweep records the higher-colour sums, next forward sweep streams half)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_au.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_au.log
run() { echo "== $1 $2" >> gpurun_out/ab_au.log; env $1 timeout 400 python bench.py --config $2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/ab_au.err | tail -1 >> gpurun_out/ab_au.log; }
run "IETI_USWEEP=0" C5
run "IETI_NONE=1" C5
run "IETI_USWEEP=0" C4
run "IETI_NONE=1" C4
run "IETI_USWEEP=0" C3
run "IETI_NONE=1" C3
echo done
