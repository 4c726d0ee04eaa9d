#!/bin/bash
# pass ar: programmatic dependent launch of the transfer kernels (IETI_PDL_TR) and of the cluster sweeps
# (IETI_PDL_CL: static prologue incl. phase 0's list / slab before the wait, dependents released in the
# last phase): bitwise + parity tests on the small configs, then A/B bench lines C4 / C3 / C2 / C1
mkdir -p gpurun_out
t=r2ar
timeout 1500 python -m pytest tests -m gpu -q -x -k "cluster_sweep_bitwise or solve_parity or vcycle_and_local or bitwise_reproducible or fused_vcycle" > gpurun_out/pytest_pdl_$t.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_pdl_$t.txt; tail -3 gpurun_out/pytest_pdl_$t.txt
for cfg in C4 C3 C2 C1; do
  for v in 00 10 01 11; do
    IETI_PDL_TR=${v:0:1} IETI_PDL_CL=${v:1:1} python bench.py --config $cfg --no-cpu-baseline --no-e2e --steps 10 --warmup 3 > gpurun_out/ab_pdl_${cfg}_$v.json 2>/dev/null
    python - gpurun_out/ab_pdl_${cfg}_$v.json $cfg $v <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[2], "TR,CL =", sys.argv[3], "it/s", round(d["value"], 2), "its", d["config"].get("pcg_iterations_per_solve"))
except Exception as e:
    print(sys.argv[2], sys.argv[3], "FAILED", e)
PY
  done
done | tee gpurun_out/ab_pdl_summary_$t.txt
find gpurun_out -type f -size +20M -delete
