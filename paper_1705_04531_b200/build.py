"""Build libieti.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
import concurrent.futures as cf
import hashlib
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
# IETI_DEBUG_BOUNDS=1: bounds-checked stencil gathers (trap on a read outside the level pool); the
# flag is part of the build info, so a debug library is never mistaken for the product
DEBUG_BOUNDS = os.environ.get("IETI_DEBUG_BOUNDS") == "1"
FLAGS = (["-DIETI_DEBUG_BOUNDS"] if DEBUG_BOUNDS else []) + [
         "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
         "-I" + os.path.join(HERE, "..", "include"), "-I" + os.path.join(NCCL_DIR, "include"),
         '-DIETI_NCCL_PATH="%s"' % os.path.join(NCCL_DIR, "lib", "libnccl.so.2")]
SOURCES = ["kernels_mg.cu", "kernels_sweep.cu", "kernels_asm.cu", "kernels_ieti.cu", "kernels_basis.cu", "kernels_direct.cu",
           "solver.cu",
           "host_topology.cpp", "partition.cpp", "comm.cpp"]


def _stale(obj, deps):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def source_files():
    """Every file the library is compiled from (sources, csrc headers, the public header, build.py)."""
    inc = os.path.join(HERE, "..", "include")
    files = [os.path.join(CSRC, f) for f in SOURCES]
    files += sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh")))
    files += sorted(os.path.join(inc, f) for f in os.listdir(inc) if f.endswith(".h"))
    return files + [os.path.abspath(__file__)]


def source_hash():
    """sha256 over the library's sources (name + bytes); compiled into libieti.so (ieti_build_info)
    so that every run can prove which sources it executed."""
    h = hashlib.sha256()
    for f in source_files():
        h.update(os.path.basename(f).encode())
        with open(f, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def build(verbose=False, force=False):
    os.makedirs(BUILD, exist_ok=True)
    # every header under csrc/ and include/ is a dependency of every object (layout.cuh defines the
    # device structs shared by the kernels and the host code)
    headers = sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh")))
    inc = os.path.join(HERE, "..", "include")
    headers += sorted(os.path.join(inc, f) for f in os.listdir(inc) if f.endswith(".h"))
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
    # build provenance: the source hash as a compiled-in string
    sh = source_hash()
    info_src = os.path.join(BUILD, "build_info.cpp")
    info_obj = info_src + ".o"
    old = open(info_src).read() if os.path.exists(info_src) else ""
    text = ('extern "C" const char *ieti_build_info(void) { return "src=%s arch=sm_100a nvcc_flags=%s%s"; }\n'
            % (sh, " ".join(f for f in FLAGS if f.startswith("-O") or f == "-lineinfo"),
               " debug_bounds" if DEBUG_BOUNDS else ""))
    relink = force or bool(jobs) or not os.path.exists(LIB)
    if text != old or not os.path.exists(info_obj):
        with open(info_src, "w") as fh:
            fh.write(text)
        r = subprocess.run(["g++", "-O2", "-fPIC", "-c", info_src, "-o", info_obj], capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("build_info compile failed")
        relink = True
    objs.append(info_obj)
    if relink:
        cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs + ["-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link failed")
    return LIB


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    print(LIB)
