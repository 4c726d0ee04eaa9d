"""Build libieti.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libieti.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NCCL_DIR = None
for _sp in [os.path.dirname(os.path.dirname(os.__file__)) + "/site-packages"] + sys.path:
    _d = os.path.join(_sp, "nvidia", "nccl")
    if os.path.exists(os.path.join(_d, "include", "nccl.h")):
        NCCL_DIR = _d
        break
if NCCL_DIR is None:
    raise RuntimeError("nccl.h not found (nvidia/nccl wheel)")
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
         "-I" + os.path.join(HERE, "..", "include"), "-I" + os.path.join(NCCL_DIR, "include"),
         '-DIETI_NCCL_PATH="%s"' % os.path.join(NCCL_DIR, "lib", "libnccl.so.2")]
SOURCES = ["kernels_mg.cu", "kernels_asm.cu", "kernels_ieti.cu", "kernels_basis.cu", "solver.cu",
           "host_topology.cpp", "partition.cpp", "comm.cpp"]


def _stale(obj, deps):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose=False, force=False):
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(CSRC, "internal.h"), os.path.join(HERE, "..", "include", "ieti.h")]
    jobs = []
    objs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            cmd = [NVCC] + ARCH + FLAGS + ["-c", s, "-o", o]
            if src.endswith(".cu"):
                cmd[1:1] = ["-Xptxas", "-v"] if verbose else []
            jobs.append(cmd)

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        return cmd, r

    with cf.ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        for cmd, r in ex.map(run, jobs):
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError("nvcc failed: " + " ".join(cmd))
            if verbose and r.stderr:
                sys.stderr.write(r.stderr)
    if force or jobs or not os.path.exists(LIB):
        cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs + ["-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link failed")
    return LIB


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    print(LIB)
