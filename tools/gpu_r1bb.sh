#!/bin/bash
# pass bb: variant replicas re-run after the upload-ordering fix
mkdir -p gpurun_out
timeout 1500 python tools/paper_replica.py --workload E1 --grid 4,8 --variant all 64 128 256 512 > gpurun_out/replica_E1_bb.jsonl 2> gpurun_out/replica_E1_bb.err
timeout 900 python tools/paper_replica.py --workload E1 --grid 4,8 --variant MGMG,MGD 1024 >> gpurun_out/replica_E1_bb.jsonl 2>> gpurun_out/replica_E1_bb.err
timeout 1500 python tools/paper_replica.py --workload E2 --grid 4,8,4 --variant all 4 8 16 > gpurun_out/replica_E2_bb.jsonl 2> gpurun_out/replica_E2_bb.err
timeout 900 python tools/paper_replica.py --workload E2 --grid 4,8,4 --variant MGMG,MGD 32 >> gpurun_out/replica_E2_bb.jsonl 2>> gpurun_out/replica_E2_bb.err
timeout 900 python tools/paper_replica.py --workload E2 --grid 4,8,4 --p 4 --variant all 4 8 > gpurun_out/replica_E2p4_bb.jsonl 2> gpurun_out/replica_E2p4_bb.err
echo done
