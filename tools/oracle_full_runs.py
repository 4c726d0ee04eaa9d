"""Whole-solve CPU oracle timings (the cpu baseline of SURVEY 8(d) / BASELINE.md, run on the GPU
box's host cores): for each config, setup, d^, the PCG loop and the recovery timed separately,
(a) one process with OMP_NUM_THREADS=1 and (b) the patch-sharded oracle on all cores (fixed-cycle
configs; oracle/sharded.py, same arithmetic).  Calls only oracle/ and workloads/.

usage: OMP_NUM_THREADS=1 python tools/oracle_full_runs.py C1 C2 C3 C4 [--out file.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.ieti import IetiOracle            # noqa: E402
from oracle.sharded import ShardedIetiOracle  # noqa: E402
from workloads import make_workload           # noqa: E402


def timed(orc, wl):
    t0 = time.perf_counter()
    orc.rhs_d()
    t_d = time.perf_counter() - t0
    t0 = time.perf_counter()
    res = orc.solve(tol=wl.pcg_tol)
    t_solve = time.perf_counter() - t0
    t0 = time.perf_counter()
    orc.recover(res.lam)
    t_rec = time.perf_counter() - t0
    t_loop = max(0.0, t_solve - t_d - t_rec)
    return dict(iters=res.iters, rel_res=res.rel_res, t_d_s=t_d, t_loop_s=t_loop, t_recovery_s=t_rec,
                t_solve_s=t_solve, it_per_s=res.iters / t_loop if t_loop > 0 else None)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--out", default=None)
    ap.add_argument("--workers", type=int, default=len(os.sched_getaffinity(0)))
    a = ap.parse_args()
    facts = {"cores": len(os.sched_getaffinity(0)), "omp_num_threads": os.environ.get("OMP_NUM_THREADS")}
    for line in open("/proc/cpuinfo"):
        if line.startswith("model name"):
            facts["cpu_model"] = line.split(":", 1)[1].strip()
            break
    for line in open("/proc/meminfo"):
        if line.startswith("MemTotal"):
            facts["ram_gb"] = round(int(line.split()[1]) / 2 ** 20, 1)
    out = {"host": facts, "runs": []}
    for name in a.configs:
        wl = make_workload(name)
        t0 = time.perf_counter()
        orc = IetiOracle(wl)
        rec = {"config": name, "mode": "one process", "setup_s": time.perf_counter() - t0}
        rec.update(timed(orc, wl))
        out["runs"].append(rec)
        print(json.dumps(rec), flush=True)
        if wl.local_mode == 0:
            topo = orc.topo
            del orc
            t0 = time.perf_counter()
            sh = ShardedIetiOracle(wl, workers=a.workers, basis="kkt", topo=topo)
            rec = {"config": name, "mode": f"patch-sharded, {a.workers} processes",
                   "setup_s": time.perf_counter() - t0}
            rec.update(timed(sh, wl))
            sh.close()
            out["runs"].append(rec)
            print(json.dumps(rec), flush=True)
    if a.out:
        json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
