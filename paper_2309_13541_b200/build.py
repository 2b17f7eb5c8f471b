"""Build the native pieces in-tree (the .so files travel to the GPU box).

  paper_2309_13541_b200/_a2a_exec.so   executor: C++ plan builder + sm_100a kernels
                                       (nvcc -gencode arch=compute_100a,code=sm_100a)
  oracle/_build/liboracle_replay.so     CPU oracle restatement in C (test/bench only)

Usage: python -m paper_2309_13541_b200.build [--force]
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "_a2a_exec.so")
ORACLE_SRC = os.path.join(ROOT, "oracle", "replay_bytes.c")
ORACLE_LIB = os.path.join(ROOT, "oracle", "_build", "liboracle_replay.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(out, srcs):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(s) > t for s in srcs)


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def build_native(force: bool = False, verbose: bool = True) -> str:
    srcs = [os.path.join(CSRC, f) for f in ("a2a_plan.cpp", "a2a_io.cpp", "a2a_sim.cpp", "a2a_exec.cu")]
    deps = srcs + [os.path.join(CSRC, "a2a_internal.h"), os.path.join(INCLUDE, "a2a_exec.h")]
    if force or _stale(LIB, deps):
        tmp = LIB + ".tmp"
        _run([_nvcc(), *ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xptxas", "-v",
              "-Xcompiler", "-fPIC,-O3", "-shared", "-I", INCLUDE, "-I", CSRC,
              *srcs, "-lz", "-o", tmp], verbose)
        os.replace(tmp, LIB)
    return LIB


def build_oracle(force: bool = False, verbose: bool = True) -> str | None:
    if not os.path.exists(ORACLE_SRC):
        return None
    os.makedirs(os.path.dirname(ORACLE_LIB), exist_ok=True)
    if force or _stale(ORACLE_LIB, [ORACLE_SRC]):
        tmp = ORACLE_LIB + ".tmp"
        _run(["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
              ORACLE_SRC, "-o", tmp], verbose)
        os.replace(tmp, ORACLE_LIB)
    return ORACLE_LIB


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    force = "--force" in argv
    print(build_native(force))
    print(build_oracle(force))


if __name__ == "__main__":
    main()
