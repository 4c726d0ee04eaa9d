#!/bin/bash
mkdir -p gpurun_out
for k in 1 2 3; do timeout 300 python tools/determinism2.py C3 >> gpurun_out/det_ax.log 2>&1; done
echo done
