"""Build libhlq_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2406_15102_b200.build [--verbose]

The library is a plain C-ABI shared object (no torch / Python headers), so it
travels to the GPU box as a single file next to this module.  Numerics flags
are part of the bit-exact contract: no --use_fast_math, IEEE division and
square root, denormals preserved (nvcc defaults, spelled out explicitly).
"""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libhlq_b200.so")
SOURCES = ["hlq_transform.cu", "hlq_transform_fallback.cu", "hlq_conv.cu", "hlq_gemm.cu", "hlq_weights.cu",
           "hlq_stochastic.cu", "hlq_baselines.cu", "hlq_acbp.cu", "hlq_capi.cu"]
HEADERS = ["hlq_ptx.cuh", "hlq_quant.cuh", "hlq_philox.cuh", "hlq_internal.h", os.path.join("..", "..", "include", "hlq_b200.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-ftz=false", "-prec-div=true", "-prec-sqrt=true", "-fmad=true",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-cudart", "static",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [__file__]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    # translation units compile in parallel; objects are kept (git-ignored) so a
    # rebuild only recompiles sources newer than their object or any header
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    hdr_t = max(os.path.getmtime(os.path.join(CSRC, h)) for h in HEADERS
                if os.path.exists(os.path.join(CSRC, h)))
    hdr_t = max(hdr_t, os.path.getmtime(__file__))
    objs, procs = [], []
    for src in SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        objs.append(obj)
        srcp = os.path.join(CSRC, src)
        if (not force and os.path.exists(obj) and os.path.getmtime(obj) > os.path.getmtime(srcp)
                and os.path.getmtime(obj) > hdr_t):
            continue
        cmd = [nvcc(), *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-c", srcp, "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd))
        procs.append((src, subprocess.Popen(cmd)))
    for src, p in procs:
        if p.wait() != 0:
            raise subprocess.CalledProcessError(p.returncode, f"nvcc {src}")
    # the driver API (cuTensorMapEncodeTiled) is resolved at run time through
    # cudaGetDriverEntryPoint, so there is no link-time libcuda dependency
    cmd = [nvcc(), *NVCC_FLAGS, "-shared", *objs, "-o", LIB]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    return LIB


def build_trace() -> str:
    """Development build with -DHLQ_TR_TRACE (per-CTA globaltimer stamps of the
    fused transform, tools/tr_timeline.py) into libhlq_b200_trace.so."""
    objdir = os.path.join(HERE, "build_trace")
    os.makedirs(objdir, exist_ok=True)
    out = os.path.join(HERE, "libhlq_b200_trace.so")
    objs, procs = [], []
    for src in SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        objs.append(obj)
        procs.append(subprocess.Popen([nvcc(), *NVCC_FLAGS, "-DHLQ_TR_TRACE", "-I", os.path.join(ROOT, "include"),
                                       "-c", os.path.join(CSRC, src), "-o", obj]))
    for p in procs:
        if p.wait() != 0:
            raise subprocess.CalledProcessError(p.returncode, "nvcc (trace build)")
    subprocess.run([nvcc(), *NVCC_FLAGS, "-shared", *objs, "-o", out], check=True)
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--trace", action="store_true", help="also build libhlq_b200_trace.so (-DHLQ_TR_TRACE)")
    a = ap.parse_args()
    print(build(force=a.force or a.verbose, verbose=a.verbose))
    if a.trace:
        print(build_trace())
    sys.exit(0)
