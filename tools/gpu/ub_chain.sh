#!/bin/bash
# ubench: cost of a chain of dependent descriptor loads at block start (library: blocks->probs->grids->cinfo)
mkdir -p gpurun_out
cd tools/ubench && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o sweep sweep.cu && \
timeout 600 ./sweep 256 10 "chain cord" > ../../gpurun_out/ub_chain.txt 2>&1; echo "rc=$?"; cat ../../gpurun_out/ub_chain.txt
