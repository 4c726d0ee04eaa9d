#!/bin/bash
# pass ba: final round-1 sweep after the U-sweep and the upload-ordering fix
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --durations=5 > gpurun_out/pytest_gpu_ba.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_ba.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_ba.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_ba.log
for C in C4 C3 C2 C1; do
  timeout 600 python bench.py --config $C --steps 5 --warmup 3 > gpurun_out/bench_${C}_ba.json 2> gpurun_out/bench_${C}_ba.err
done
( time timeout 1200 python bench.py ) > gpurun_out/bench_default_ba.json 2> gpurun_out/bench_default_ba.err
timeout 400 python bench.py --config C5 --profile-iters 1 --no-e2e > gpurun_out/plain_C5_ba.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches_C5_ba.csv python bench.py --config C5 --profile-iters 1 --no-e2e > gpurun_out/ncu_list_C5_ba.log 2>&1
timeout 1500 ncu --set full --cache-control none --clock-control none --import-source on --profile-from-start off \
  --kernel-name-base demangled -k "regex:k_stencil<.int.3, .int.3, .int.1, .int.[067]" --launch-skip 64 -c 3 -o gpurun_out/sgs_C5_ba \
  python bench.py --config C5 --profile-iters 1 --no-e2e > gpurun_out/ncu_full_C5_ba.log 2>&1
echo done
