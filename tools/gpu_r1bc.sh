#!/bin/bash
mkdir -p gpurun_out
IETI_VERBOSE=1 timeout 600 python bench.py --config C5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/verbose_bc.json 2> gpurun_out/verbose_bc.err
echo done
