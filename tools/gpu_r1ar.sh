#!/bin/bash
# pass ar: final round-1 evidence: full GPU suite, smoke, default bench line, ncu --set full of the finest SGS phase
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --durations=8 > gpurun_out/pytest_gpu_ar.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_ar.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_ar.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_ar.log
( time timeout 1200 python bench.py ) > gpurun_out/bench_default_ar.json 2> gpurun_out/bench_default_ar.err
timeout 1500 ncu --set full --cache-control none --clock-control none --import-source on --profile-from-start off \
  --kernel-name-base demangled -k "regex:k_stencil<3, 3, 1, 0" --launch-skip 64 -c 2 -o gpurun_out/sgs_C5_ar \
  python bench.py --config C5 --profile-iters 1 --no-e2e > gpurun_out/ncu_full_C5_ar.log 2>&1
echo done
