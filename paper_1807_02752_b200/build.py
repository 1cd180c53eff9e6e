"""Builds the in-tree sm_100a library liblanekit_b200.so with nvcc.

The shared object travels with the repo snapshot to the GPU box (it is
git-ignored, not gpurun-ignored). Flags:
  -gencode arch=compute_100a,code=sm_100a  B200 only, no multi-arch fallback
  --fmad=false                             no FMA contraction: bit-exact FP64
  -Xcompiler -ffp-contract=off             same for the host-built tables
  -lineinfo                                ncu source view
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "liblanekit_b200.so"
SOURCES = ["lk_api.cu", "lk_kernels.cu", "lk_fastpath.cu", "lk_stereo.cu", "synth.cpp"]
HEADERS = ["lk_device.cuh", "lk_fit.cuh", "lk_kernels.h", "../../include/lanekit_b200.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC,-ffp-contract=off",
    "-shared", "-cudart", "static",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (Path(cand).exists() or cand == "nvcc"):
            return cand
    return "nvcc"


def stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + [CSRC / h for h in HEADERS]
    return any(p.stat().st_mtime > t for p in deps if p.exists())


def build(force: bool = False, verbose: bool = False) -> Path:
    if force or stale():
        cmd = [nvcc(), *NVCC_FLAGS, *[str(CSRC / s) for s in SOURCES], "-o", str(LIB)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True, cwd=str(CSRC))
    build_cli(force, verbose)
    return LIB


CLI = PKG / "lanedet_gpu"


def build_cli(force: bool = False, verbose: bool = False) -> Path:
    """lanedet_gpu: the reference's lanedet CLI over the C-ABI (host C++ + zlib)."""
    src = CSRC / "lanedet_gpu.cpp"
    if not force and CLI.exists() and CLI.stat().st_mtime >= max(
            src.stat().st_mtime, LIB.stat().st_mtime):
        return CLI
    cmd = [os.environ.get("CXX", "g++"), "-std=c++17", "-O2", "-Wall", "-pthread", str(src),
           f"-L{PKG}", "-llanekit_b200", "-lz", "-Wl,-rpath,$ORIGIN", "-o", str(CLI)]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True, cwd=str(CSRC))
    return CLI


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
