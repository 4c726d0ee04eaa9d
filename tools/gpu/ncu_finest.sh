#!/bin/bash
# ncu --set full of mid-sweep finest-level colour-SGS launches of C5 (full sweeps, modes 7 and 0) on the current
# build; only the text summaries come back.  usage: bash tools/gpu/ncu_finest.sh <tag>
mkdir -p gpurun_out
t=${1:-x}
CMD="python bench.py --config C5 --profile-iters 1 --no-cpu-baseline"
for m in 7 0; do
  ncu --set full --clock-control none --import-source on --profile-from-start off --kernel-name-base demangled \
      -k "regex:k_stencil<\(int\)3, \(int\)3, \(int\)1, \(int\)$m," -s 90 -c 3 -o gpurun_out/ncu_sgs${m}_$t -f $CMD > gpurun_out/ncu_sgs${m}_$t.log 2>&1
  echo "ncu mode $m rc=$?"
  python tools/ncu_summary.py full gpurun_out/ncu_sgs${m}_$t.ncu-rep > gpurun_out/ncu_sgs${m}_$t.txt 2>&1
  rm -f gpurun_out/ncu_sgs${m}_$t.ncu-rep
done
find gpurun_out -type f -size +20M -delete
