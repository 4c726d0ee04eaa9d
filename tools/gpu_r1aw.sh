#!/bin/bash
# pass aw: determinism probe (C3, C4, C1), twice each in separate processes, with and without PDL / U-sweep
mkdir -p gpurun_out
for C in C3 C4 C1; do
  for k in 1 2; do timeout 300 python tools/determinism.py $C >> gpurun_out/det_aw.log 2>&1; done
done
for k in 1 2; do IETI_PDL=0 timeout 300 python tools/determinism.py C3 >> gpurun_out/det_aw.log 2>&1; done
for k in 1 2; do IETI_USWEEP=0 timeout 300 python tools/determinism.py C3 >> gpurun_out/det_aw.log 2>&1; done
for k in 1 2; do IETI_PF=0 timeout 300 python tools/determinism.py C3 >> gpurun_out/det_aw.log 2>&1; done
echo done
