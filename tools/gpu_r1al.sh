#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/probe_inner.py E2 4 4 4,8,4 > gpurun_out/probe_al.log 2>&1
timeout 300 python tools/probe_inner.py E2 8 4 4,8,4 >> gpurun_out/probe_al.log 2>&1
timeout 300 python tools/probe_inner.py E2 8 2 4,8,4 >> gpurun_out/probe_al.log 2>&1
echo done
