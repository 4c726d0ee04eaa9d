#!/bin/bash
# pass aq: 4-deep / 16-CTA variant on the tpr-8 levels (C5, C4)
mkdir -p gpurun_out
run() { echo "== $1 $2" >> gpurun_out/ab_aq.log; env $1 timeout 400 python bench.py --config $2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/ab_aq.err | tail -1 >> gpurun_out/ab_aq.log; }
run "IETI_NONE=1" C5
run "IETI_BATCH=4" C5
run "IETI_NONE=1" C4
run "IETI_BATCH=4" C4
run "IETI_NONE=1" C3
run "IETI_BATCH=4" C3
timeout 300 python -m pytest tests -m gpu -q -k "C4s or C5s" > gpurun_out/pytest_gpu_aq.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_aq.log
IETI_BATCH=4 timeout 300 python -m pytest tests -m gpu -q -k "C4s or C5s" >> gpurun_out/pytest_gpu_aq.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_aq.log
echo done
