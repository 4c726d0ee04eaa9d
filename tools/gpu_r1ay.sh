#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/determinism3.py dump /tmp/stA.npy > gpurun_out/det_ay.log 2>&1
timeout 300 python tools/determinism3.py dump /tmp/stB.npy >> gpurun_out/det_ay.log 2>&1
timeout 300 python tools/determinism3.py cmp /tmp/stA.npy /tmp/stB.npy >> gpurun_out/det_ay.log 2>&1
timeout 300 python tools/determinism3.py cmp /tmp/stA.npy.N.npy /tmp/stB.npy.N.npy >> gpurun_out/det_ay.log 2>&1
echo done
