#!/bin/bash
# is the in-situ gap to the microbenchmark the power cap? the same sweep timed for ~4 s (sustained)
# vs 50 ms (burst), and a sustained device copy, with the SM clock sampled during each
mkdir -p gpurun_out
cd tools/ubench && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o sweep sweep.cu && cd ../..
clk() { nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv,noheader -lms 200 > gpurun_out/clk_$1.txt & echo $!; }
p=$(clk burst); tools/ubench/sweep 256 10 "cord" | grep -v ORD; kill $p
p=$(clk sustained); tools/ubench/sweep 256 800 "cord" | grep -v ORD; kill $p
p=$(clk copy); python - <<'PY'
import torch, time
a = torch.empty(2 << 30, dtype=torch.uint8, device="cuda"); b = torch.empty_like(a)
for n in (10, 2000):
    torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): b.copy_(a)
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3
    print(f"copy 2 GiB x {n}: {2 * a.numel() * n / t / 1e9:.1f} GB/s over {t:.2f} s")
PY
kill $p
for f in burst sustained copy; do echo "$f: $(sort -t, -k1 -n gpurun_out/clk_$f.txt | awk -F, '{print $1}' | sort -n | awk '{a[NR]=$1} END {print "sm MHz median", a[int(NR/2)+1], "min", a[1], "max", a[NR]}')"; sort gpurun_out/clk_$f.txt | awk -F, '{print $3}' | sort | uniq -c | head -3; done
