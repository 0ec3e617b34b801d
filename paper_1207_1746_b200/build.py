"""Build libgscl.so in-tree for sm_100a with nvcc (no JIT cache, no torch
extension machinery): each .cu -> .o, then one shared library linked against
the static CUDA runtime and the NCCL that ships with PyTorch's wheels.

GSCL_ABLATIONS=1 (or build(ablations=True)) builds libgscl_ablations.so
instead: the same library plus the measured-and-rejected kernel designs and
their gscl_set_option knobs (sweep_impl, variant, zchunks, sched, stages,
l2promo, zalt).  The product library never contains them; load the ablation
build with GSCL_LIB=<path> (gscl.py)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libgscl.so")
BUILD_ABL = os.path.join(HERE, "build_ablations")
LIB_ABL = os.path.join(HERE, "libgscl_ablations.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-fmad=false",
                  "-ftz=false", "-prec-div=true", "-prec-sqrt=true", "-Xptxas", "-v",
                  "--expt-relaxed-constexpr"]


def nccl_dirs():
    site = sysconfig.get_paths()["purelib"]
    base = os.path.join(site, "nvidia", "nccl")
    inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
    if not os.path.exists(os.path.join(inc, "nccl.h")):
        raise RuntimeError(f"nccl.h not found under {inc}")
    return inc, lib


def build(force: bool = False, verbose: bool = False, ablations: bool | None = None) -> str:
    if ablations is None:
        ablations = os.environ.get("GSCL_ABLATIONS", "0") not in ("", "0")
    bdir, lib = (BUILD_ABL, LIB_ABL) if ablations else (BUILD, LIB)
    flags = NVFLAGS + (["-DGSCL_ABLATIONS=1"] if ablations else [])
    inc, nlib = nccl_dirs()
    os.makedirs(bdir, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    deps = srcs + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        [os.path.join(ROOT, "include", "gscl.h"), os.path.abspath(__file__)]
    newest = max(os.path.getmtime(d) for d in deps)
    if not force and os.path.exists(lib) and os.path.getmtime(lib) >= newest:
        return lib
    # headers and flags are shared by every translation unit; a source whose
    # object is newer than it and than every shared dependency is not recompiled
    shared = max(os.path.getmtime(d) for d in deps if not d.endswith(".cu"))
    objs = []
    procs = []
    for s in srcs:
        o = os.path.join(bdir, os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        if not force and os.path.exists(o) and os.path.getmtime(o) >= max(shared, os.path.getmtime(s)):
            continue
        cmd = [NVCC] + flags + ["-I", inc, "-I", os.path.join(ROOT, "include"), "-c", s, "-o", o]
        log = open(o + ".log", "w")
        procs.append((subprocess.Popen(cmd, stdout=log, stderr=subprocess.STDOUT), o, cmd))
    for p, o, cmd in procs:
        if p.wait() != 0:
            sys.stderr.write(open(o + ".log").read())
            raise RuntimeError("nvcc failed: " + " ".join(cmd))
        if verbose:
            sys.stdout.write(open(o + ".log").read())
    tmp = lib + f".tmp{os.getpid()}"
    link = [NVCC] + ARCH + ["-shared", "-o", tmp] + objs + \
        ["-L", nlib, "-l:libnccl.so.2", "-Xlinker", f"-rpath={nlib}", "-cudart", "static"]
    subprocess.run(link, check=True)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv,
                ablations=True if "--ablations" in sys.argv else None))
