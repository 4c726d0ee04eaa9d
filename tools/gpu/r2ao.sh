#!/bin/bash
# pass ao: primal-basis PCG with converged columns masked out of the stencil kernels (IETI_BASIS_MASK):
# bitwise test, C5 setup stages with the mask off / on (+ per-chunk iteration spread), Phibar parity tests,
# C4 / C3 launch lists on the current build, per-rank proxies of C5 re-measured
mkdir -p gpurun_out
t=r2ao
timeout 1500 python -m pytest tests -m gpu -q -k "basis_mask or primal_basis or full_size" > gpurun_out/pytest_basis_$t.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_basis_$t.txt; tail -3 gpurun_out/pytest_basis_$t.txt
cat > /tmp/setup_c5.py <<'PY'
import time, sys
import paper_1705_04531_b200 as lib
from workloads import make_workload
wl = make_workload("C5")
t = time.time(); g = lib.Ieti.from_workload(wl); print("setup_s", time.time() - t, file=sys.stderr); g.close()
PY
for m in 0 1; do
  IETI_VERBOSE=1 IETI_BASIS_MASK=$m PYTHONPATH=$PWD python /tmp/setup_c5.py 2>&1 | grep -E "ieti setup|basis chunk|setup_s" > gpurun_out/setup_stages_C5_mask${m}_$t.txt
  tail -4 gpurun_out/setup_stages_C5_mask${m}_$t.txt
done
for g in 4,8,4 4,4,4 4,4,2; do
  python bench.py --config C5 --grid $g --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/proxy_C5_${g//,/x}_$t.json 2> gpurun_out/proxy_$t.err; echo "proxy $g rc=$?"
done
for cfg in C4 C3; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_${cfg}_$t.csv python bench.py --config $cfg --profile-iters 1 --no-cpu-baseline > /dev/null 2>&1
  echo "ncu $cfg rc=$?"
  python tools/ncu_summary.py launches gpurun_out/launches_${cfg}_$t.csv > gpurun_out/launches_${cfg}_$t.txt 2>&1; rm -f gpurun_out/launches_${cfg}_$t.csv
done
