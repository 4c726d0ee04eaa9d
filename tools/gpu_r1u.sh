#!/bin/bash
# pass u: persisting-L2 window for the finest x (A/B), ncu of the finest MODE-0 phase (fixed regex)
mkdir -p gpurun_out
python - > gpurun_out/l2attrs.txt <<'PY'
import torch
print(torch.cuda.get_device_properties(0))
PY
for L in 1 0; do
  IETI_L2P=$L timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5_u_l2p$L.json 2> gpurun_out/bench_C5_u_l2p$L.err
done
IETI_L2P=1 timeout 600 python -m pytest tests -m gpu -q -k "C5s or C4s" > gpurun_out/pytest_gpu_u.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_u.log
timeout 1500 ncu --set full --cache-control none --clock-control none --import-source on --profile-from-start off \
  --kernel-name-base demangled -k "regex:k_stencil<.int.3, .int.3, .int.1, .int.0>" --launch-skip 64 -c 3 -o gpurun_out/sgs_C5_u \
  python bench.py --config C5 --profile-iters 1 --no-e2e > gpurun_out/ncu_full_C5_u.log 2>&1
echo done
