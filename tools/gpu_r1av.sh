#!/bin/bash
# pass av: repeat the mode-6/7 A/B on C3, C2, C1 (and C5 once more)
mkdir -p gpurun_out
run() { echo "== $1 $2" >> gpurun_out/ab_av.log; env $1 timeout 400 python bench.py --config $2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/ab_av.err | tail -1 >> gpurun_out/ab_av.log; }
for C in C3 C2 C1; do
  run "IETI_USWEEP=0" $C; run "IETI_NONE=1" $C; run "IETI_USWEEP=0" $C; run "IETI_NONE=1" $C
done
run "IETI_NONE=1" C5
run "IETI_USWEEP=0" C5
echo done
