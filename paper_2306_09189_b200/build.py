"""Builds libfheconv.so in-tree with nvcc for sm_100a (B200).

The shared library exports the C ABI of include/fheconv.h. It is built
in-tree (not into a JIT cache) so it travels to the GPU box with the repo
snapshot. Host code is compiled with -ffp-contract=off because the host
encoder must reproduce the CPU golden model's double operations exactly.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libfheconv.so")
SOURCES = ["ntt.cu", "kernels.cu", "matvec.cu", "fheconv.cu"]
HEADERS = ["kernels.cuh", "modarith.cuh", "host_math.hpp", "cdt_table.h"]

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
    "-Xptxas", "-O3",
    # no -split-compile: it halves the build time but makes code generation depend on how a
    # translation unit's kernels are partitioned (k_pt_matvec2 a third slower, k_bsgs_tma +-2 %
    # as kernels move between files; profiles/ab_r02_split_compile.txt)
    "-I", os.path.join(ROOT, "include"),
]


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "fheconv.h")]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    objs = []
    jobs = []  # the translation units compile side by side (kernels.cu alone is ~2 minutes)
    hdr = [os.path.join(CSRC, f) for f in HEADERS] + [os.path.join(ROOT, "include", "fheconv.h")]
    for src in SOURCES:
        obj = os.path.join(CSRC, src.replace(".cu", ".o"))
        deps = [os.path.join(CSRC, src)] + hdr
        objs.append(obj)
        if not force and os.path.exists(obj) and all(os.path.getmtime(d) <= os.path.getmtime(obj) for d in deps
                                                     if os.path.exists(d)):
            continue
        cmd = [_nvcc(), *NVCC_FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), file=sys.stderr)
        jobs.append((cmd, subprocess.Popen(cmd)))
    failed = [cmd for cmd, pr in jobs if pr.wait() != 0]
    if failed:
        raise subprocess.CalledProcessError(1, failed[0])
    tmp = LIB + ".tmp"
    subprocess.run([_nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp, *objs],
                   check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
