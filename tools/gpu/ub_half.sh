#!/bin/bash
# ubench: half-coefficient sweep (the library's modes 4/6) vs the full sweep, concurrent groups
mkdir -p gpurun_out
cd tools/ubench && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o sweep sweep.cu && \
timeout 600 ./sweep 256 10 "half cord" > ../../gpurun_out/ub_half.txt 2>&1; echo "rc=$?"; grep -v ORD ../../gpurun_out/ub_half.txt
