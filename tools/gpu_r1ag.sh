#!/bin/bash
# pass ag: Table-2 replica (E2: 3D annulus 4x8x4, p=2, edge averages, MG-MG), two orientations
mkdir -p gpurun_out
timeout 1800 python tools/paper_replica.py --workload E2 4 8 16 32 > gpurun_out/paper_replica_ag_E2.jsonl 2> gpurun_out/paper_replica_ag_E2.err
timeout 1200 python tools/paper_replica.py --workload E2 --grid 4,4,8 4 8 16 > gpurun_out/paper_replica_ag_E2b.jsonl 2> gpurun_out/paper_replica_ag_E2b.err
echo done
