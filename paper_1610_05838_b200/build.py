"""Build libmf.so (CUDA for sm_100a) in-tree with nvcc.  No torch types cross the ABI."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libmf.so")
SOURCES = ["mf_api.cu", "mf_kernels.cu", "mf_wavefront.cu", "mf_partition.cu", "mf_stream.cu", "mf_outcore.cu",
           "mf_flow.cu"]
HEADERS = ["mf_ctx.h", "mf_kernels.cuh", "sgd_core.cuh", "mf_host_util.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
         "-Xptxas", "-v", "-I", os.path.join(HERE, "..", "include")]


def _stale(obj, src):
    deps = [src] + [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(HERE, "..", "include", "mf.h")]
    return not os.path.exists(obj) or any(os.path.getmtime(d) > os.path.getmtime(obj) for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    objs, procs = [], []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(objdir, s.replace(".cu", ".o"))
        objs.append(obj)
        if force or _stale(obj, src):
            log = open(obj + ".log", "w")
            procs.append((s, subprocess.Popen([NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj], stdout=log,
                                              stderr=subprocess.STDOUT), obj + ".log"))
    for s, p, log in procs:
        if p.wait() != 0:
            sys.stderr.write(open(log).read())
            raise RuntimeError(f"nvcc failed on {s}")
        if verbose:
            sys.stdout.write(open(log).read())
    if procs or not os.path.exists(SO):
        subprocess.check_call([NVCC, *ARCH, "-shared", "-o", SO, *objs, "-lnccl", "-lcuda"])
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
