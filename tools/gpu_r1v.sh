#!/bin/bash
# pass v: full GPU suite incl. large-patch parity on both stencil paths; level-2 tpr / prefetch A/B;
# then compute-sanitizer memcheck of small solves
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_v.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_v.log
for T in 4 8; do for PM in 40 100; do
  IETI_TPR=$T IETI_PFMAX=$PM timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5_v_t${T}_pm$PM.json 2> gpurun_out/bench_C5_v_t${T}_pm$PM.err
done; done
timeout 900 compute-sanitizer --tool memcheck --leak-check none python tools/sanitize_small.py > gpurun_out/memcheck_v.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/memcheck_v.log
echo done
