#!/bin/bash
# pass aj: NEXT-3 test, then variant replicas (E1 p=2 4x8, E2 p=2 4x8x4)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "next3" > gpurun_out/pytest_gpu_aj.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_aj.log
timeout 1500 python tools/paper_replica.py --workload E1 --grid 4,8 --variant all 64 128 256 512 > gpurun_out/replica_E1_variants.jsonl 2> gpurun_out/replica_E1_variants.err
timeout 1500 python tools/paper_replica.py --workload E2 --grid 4,8,4 --variant all 4 8 16 > gpurun_out/replica_E2_variants.jsonl 2> gpurun_out/replica_E2_variants.err
timeout 900 python tools/paper_replica.py --workload E2 --grid 4,8,4 --p 4 --variant all 4 8 > gpurun_out/replica_E2p4_variants.jsonl 2> gpurun_out/replica_E2p4_variants.err
echo done
