"""Build libcks.so in-tree with nvcc for sm_100a (no GPU needed)."""
from __future__ import annotations

import fcntl
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
# CKS_EXPERIMENTS=1: the experiments build (environment knobs for tools/
# sweeps, debug timeline) goes to its own file; the production libcks.so has none
EXPERIMENTS = os.environ.get("CKS_EXPERIMENTS") == "1"
LIB = os.path.join(PKG, "libcks_exp.so" if EXPERIMENTS else "libcks.so")
SOURCES = [os.path.join(CSRC, "cks_api.cu"), os.path.join(CSRC, "cks_plan.cpp")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("cks_plan.h", "kernels/ptx.cuh", "kernels/igemm.cuh",
                                                  "kernels/wgrad.cuh", "kernels/aux.cuh", "kernels/narrow.cuh",
                                                  "kernels/allreduce.cuh")] + \
    [os.path.join(os.path.dirname(PKG), "include", "cks.h")]


def nvcc_path() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile libcks.so in-tree.  Safe under concurrent callers (every torchrun
    rank calls this): an exclusive file lock serialises them, the first one
    compiles into a per-process temporary and renames it into place, the
    others then see an up-to-date library and return."""
    if not force and not needs_build():
        return LIB
    with open(LIB + ".lock", "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        try:
            if not force and not needs_build():  # another process built it meanwhile
                return LIB
            tmp = f"{LIB}.{os.getpid()}.tmp"
            cmd = [nvcc_path(), "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                   "-Xcompiler", "-fPIC", "-shared", "-o", tmp] + (["-DCKS_EXPERIMENTS"] if EXPERIMENTS else []) + SOURCES
            if EXPERIMENTS and os.environ.get("CKS_NVCC_DEFS"):  # compile-time variants (experiments build only)
                cmd += os.environ["CKS_NVCC_DEFS"].split()
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
                print(" ".join(cmd), file=sys.stderr)
            try:
                subprocess.run(cmd, check=True)
                os.replace(tmp, LIB)
            finally:
                if os.path.exists(tmp):
                    os.remove(tmp)
        finally:
            fcntl.flock(lk, fcntl.LOCK_UN)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
