#!/bin/bash
# pass as: final verification of HEAD with the transfer kernels launched programmatically (IETI_PDL_TR): GPU suite with
# the parity log, smoke, default bench line + reference arm, bench lines of C1-C4, C5 launch list + one
# --set full capture of a finest-level colour-SGS launch
mkdir -p gpurun_out
t=r2as
bash tools/gpu/parity.sh $t
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$t.txt 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/bench_C5_$t.json 2> gpurun_out/bench_C5_$t.err; echo "bench rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$t.json 2> gpurun_out/bench_ref_$t.err; echo "ref rc=$?"
for cfg in C4 C3 C2 C1; do
  python bench.py --config $cfg --no-cpu-baseline > gpurun_out/bench_${cfg}_$t.json 2> gpurun_out/bench_${cfg}_$t.err; echo "bench $cfg rc=$?"
done
CMD="python bench.py --config C5 --profile-iters 1 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --profile-from-start off --csv --log-file gpurun_out/launches_C5_$t.csv $CMD > gpurun_out/ncu_$t.log 2>&1
echo "ncu list rc=$?"
python tools/ncu_summary.py launches gpurun_out/launches_C5_$t.csv > gpurun_out/launches_C5_$t.txt 2>&1
rm -f gpurun_out/launches_C5_$t.csv
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_stencil -s 2600 -c 4 \
    -o gpurun_out/ncu_full_$t -f $CMD > gpurun_out/ncu_full_$t.log 2>&1
echo "ncu full rc=$?"
python tools/ncu_summary.py full gpurun_out/ncu_full_$t.ncu-rep > gpurun_out/ncu_full_$t.txt 2>&1
tail -2 gpurun_out/bench_C5_$t.json | cut -c1-600
rm -f gpurun_out/ncu_full_$t.ncu-rep
find gpurun_out -type f -size +20M -delete
du -sh gpurun_out
