"""In-tree build of libpbad_gpu.so (sm_100a) with nvcc; no torch JIT cache.

    python -m paper_1709_04145_b200.build

Flags that matter for parity: --fmad=false (device) and -ffp-contract=off
(host) so the only fused multiply-adds are the explicit fma() calls of the
numeric contract.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libpbad_gpu.so")
PEAK_LIB = os.path.join(PKG, "libpbad_peak.so")
BUILD = os.path.join(ROOT, "build")

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off",
              "-Xptxas", "-v"]
CUDA_SOURCES = ["pbad_kernels.cu", "pbad_chain.cu", "pbad_chain4.cu", "pbad_chain5.cu", "pbad_chain6.cu", "pbad_chain7.cu", "pbad_corr.cu", "pbad_tree.cu", "pbad_tree_lbfgs.cu", "pbad_resid.cu"]
HOST_SOURCES = ["pbad_host.cpp"]


def _run(cmd, log):
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if log is not None:
        log.write(" ".join(cmd) + "\n" + r.stdout)
    if r.returncode != 0:
        sys.stderr.write(r.stdout)
        raise RuntimeError(f"build failed: {' '.join(cmd)}")
    return r.stdout


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers.append(os.path.join(INCLUDE, "pbad_gpu.h"))
    objs, jobs = [], []
    with open(os.path.join(BUILD, "build.log"), "w") as log:
        for src in CUDA_SOURCES:
            s = os.path.join(CSRC, src)
            if not os.path.exists(s):
                continue
            o = os.path.join(BUILD, src + ".o")
            extra = [os.path.join(CSRC, "pbad_tree.cu")] if src == "pbad_tree_lbfgs.cu" else []
            if force or _stale(o, [s] + headers + extra):
                jobs.append([NVCC, *ARCH, *NVCC_FLAGS, "-I", INCLUDE, "-I", CSRC, "-c", s, "-o", o])
            objs.append(o)
        for src in HOST_SOURCES:
            s = os.path.join(CSRC, src)
            o = os.path.join(BUILD, src + ".o")
            if force or _stale(o, [s] + headers):
                jobs.append([NVCC, *ARCH, "-O2", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off,-mfma",
                             "-I", INCLUDE, "-I", CSRC, "-x", "cu", "-c", s, "-o", o])
            objs.append(o)
        # translation units compile independently (ptxas dominates): run them concurrently
        with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
            outs = list(ex.map(lambda c: _run(c, None), jobs))
        for c, out in zip(jobs, outs):
            log.write(" ".join(c) + "\n" + out)
        if force or _stale(LIB, objs):
            _run([NVCC, *ARCH, "-shared", "-o", LIB, *objs], log)
        # FP64 microbenchmark used as the roofline denominator (bench.py)
        ps = os.path.join(CSRC, "pbad_peak.cu")
        if force or _stale(PEAK_LIB, [ps]):
            _run([NVCC, *ARCH, "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", ps, "-o", PEAK_LIB], log)
    if verbose:
        print(open(os.path.join(BUILD, "build.log")).read())
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
