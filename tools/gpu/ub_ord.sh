#!/bin/bash
# ubench: offset orders for L1 reuse of the x gathers (ORD2: line-sharing offsets one batch apart)
mkdir -p gpurun_out
cd tools/ubench && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o sweep sweep.cu && \
timeout 600 ./sweep 256 6 "nb8 ord2 cord tile" > ../../gpurun_out/ub_ord.txt 2>&1; echo "rc=$?"; cat ../../gpurun_out/ub_ord.txt
