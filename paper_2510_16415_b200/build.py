"""Build libmecefo.so in-tree with nvcc for sm_100a (no JIT cache, no torch ext),
and the host-only control-plane library libmecefo_ctl.so with g++.

Usage: python -m paper_2510_16415_b200.build [--force]
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
OUT = os.path.join(HERE, "libmecefo.so")
SOURCES = ["engine.cu", "refresh.cu"]
DEPS = ["common.cuh", "host.h", "gemm.cuh", "kernels.cuh", "attention.cuh", "attention_tc.cuh", "attention_bwd_tc.cuh",
        "gemm_dual.cuh", "gemm_norm.cuh", "subspace.cuh", "ce.cuh", "refresh.cuh"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "-I", os.path.join(ROOT, "include"),
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    files = [os.path.join(CSRC, d) for d in DEPS + SOURCES if os.path.exists(os.path.join(CSRC, d))] + \
        [os.path.join(ROOT, "include", "mecefo.h")]
    return any(os.path.getmtime(f) > t for f in files)


CTL_OUT = os.path.join(HERE, "libmecefo_ctl.so")
CTL_SOURCES = [os.path.join(CSRC, "control.cpp"), os.path.join(ROOT, "include", "mecefo_ctl.h")]
CXX_FLAGS = ["-O2", "-std=c++17", "-fPIC", "-shared", "-Wall", "-I", os.path.join(ROOT, "include")]


def build_control(force: bool = False, verbose: bool = True) -> str:
    """g++ include/mecefo_ctl.h + csrc/control.cpp -> libmecefo_ctl.so (host PCG64 streams)."""
    if not force and os.path.exists(CTL_OUT) and all(os.path.getmtime(f) <= os.path.getmtime(CTL_OUT)
                                                     for f in CTL_SOURCES):
        return CTL_OUT
    cmd = [os.environ.get("CXX", "g++"), *CXX_FLAGS, "-o", CTL_OUT + ".tmp", CTL_SOURCES[0]]
    if verbose:
        print("[build]", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(CTL_OUT + ".tmp", CTL_OUT)
    return CTL_OUT


def build(force: bool = False, verbose: bool = True) -> str:
    build_control(force, verbose)
    if not force and not stale():
        return OUT
    # one translation unit per .cu, compiled in parallel, then linked
    objs, procs = [], []
    for src in [x for x in SOURCES if os.path.exists(os.path.join(CSRC, x))]:
        obj = os.path.join(CSRC, src.replace(".cu", ".o"))
        cmd = [nvcc(), *NVCC_FLAGS, "-c", "-o", obj, os.path.join(CSRC, src)]
        if verbose:
            print("[build]", " ".join(cmd), flush=True)
        procs.append(subprocess.Popen(cmd))
        objs.append(obj)
    rcs = [p.wait() for p in procs]
    if any(rcs):
        raise subprocess.CalledProcessError(max(rcs), "nvcc")
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", OUT + ".tmp", *objs]
    if verbose:
        print("[build]", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(OUT + ".tmp", OUT)
    for o in objs:
        os.remove(o)
    return OUT


def build_timing_variant(out: str = os.path.join(HERE, "libmecefo_timing.so")) -> str:
    """A second library with the timing-experiment knobs compiled in
    (-DMECEFO_TIMING_KNOBS; never loaded unless MECEFO_LIB points at it)."""
    objs, procs = [], []
    for src in [x for x in SOURCES if os.path.exists(os.path.join(CSRC, x))]:
        obj = os.path.join(CSRC, src.replace(".cu", ".timing.o"))
        procs.append(subprocess.Popen([nvcc(), *NVCC_FLAGS, "-DMECEFO_TIMING_KNOBS", "-c", "-o", obj,
                                       os.path.join(CSRC, src)]))
        objs.append(obj)
    if any(p_.wait() for p_ in procs):
        raise subprocess.CalledProcessError(1, "nvcc")
    subprocess.run([nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out, *objs], check=True)
    for o in objs:
        os.remove(o)
    return out


if __name__ == "__main__":
    if "--timing" in sys.argv:
        build_timing_variant()
    else:
        build(force="--force" in sys.argv)
