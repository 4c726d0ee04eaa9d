#!/bin/bash
# A/B: min resident blocks of the one-thread-per-row stencil kernels, 10 (48 regs) vs 8 (60 regs)
mkdir -p gpurun_out
cd paper_1705_04531_b200 && cp libieti.so libieti_kb10.so && cd ..
run() {  # tag cfg steps
  IETI_ALLOW_STALE=1 timeout 900 python bench.py --config $2 --steps $3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_kb.json 2> /dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab_kb.json')); print('$1 $2', round(d['value'],3), d['config']['pcg_iterations_per_solve'], round(d['ms_per_step'],2), 'frac', round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"
}
for rep in 1 2; do
  cp paper_1705_04531_b200/libieti_kb10.so paper_1705_04531_b200/libieti.so; run KB10 C5 5; run KB10 C3 10
  cp paper_1705_04531_b200/libieti_kb8.so paper_1705_04531_b200/libieti.so; run KB8 C5 5; run KB8 C3 10
done
cp paper_1705_04531_b200/libieti_kb10.so paper_1705_04531_b200/libieti.so
