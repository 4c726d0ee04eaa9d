#!/bin/bash
# Full-size C5 oracle dump on the GPU box's host cores (16 cores, 196 GB; ~0.4 GB of oracle
# hierarchies per patch) in the background, with the GPU parity suite running meanwhile.
mkdir -p gpurun_out
export OMP_NUM_THREADS=1
( while true; do date +%T >> gpurun_out/mem_c5.log; free -g | sed -n 2p >> gpurun_out/mem_c5.log; sleep 60; done ) &
MPID=$!
nohup timeout 4000 python tools/oracle_dump.py C5 --workers ${WORKERS:-13} --mem-gb ${MEMGB:-12} --sample 16 \
    --n-sens 0 --out gpurun_out > gpurun_out/c5_dump.log 2>&1 &
DPID=$!
bash tools/gpu/parity.sh ${TAG:-r2c}
wait $DPID
echo "dump rc=$?" >> gpurun_out/c5_dump.log
kill $MPID
tail -3 gpurun_out/c5_dump.log
