#!/bin/bash
# pass g: fused small-level V-cycle, TMA vs register fine stencils (A/B), basis projection, all configs
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_g.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_g.log
IETI_VERBOSE=1 timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5_g_tma.json 2> gpurun_out/bench_C5_g_tma.err
IETI_STENCIL=reg timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5_g_reg.json 2> gpurun_out/bench_C5_g_reg.err
for C in C4 C3 C2 C1; do
  IETI_VERBOSE=1 timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${C}_g.json 2> gpurun_out/bench_${C}_g.err
done
IETI_NO_FUSE=1 timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C4_g_nofuse.json 2> gpurun_out/bench_C4_g_nofuse.err
echo done
