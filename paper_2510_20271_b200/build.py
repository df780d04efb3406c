"""Build libecc_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2510_20271_b200.build

The library is a plain C ABI (include/ecc_b200.h) loaded with ctypes; it
travels to the GPU box with the repo snapshot (git-ignored, not
gpurun-ignored).
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libecc_b200.so"
SOURCES = ["ecc_host.cu", "ecc_discrete.cu", "ecc_fast3d.cu", "ecc_soft.cu", "ecc_fdcheck.cu"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-shared", "-Xcompiler", "-fPIC",
    # no --use_fast_math: the discrete path must not flush subnormals (FTZ)
]


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h"))
    deps.append(PKG.parent / "include" / "ecc_b200.h")
    return any(d.stat().st_mtime > t for d in deps if d.exists())


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    extra = os.environ.get("ECC_B200_NVCC_EXTRA", "").split()   # development A/B switches (-D...)
    cmd = [nvcc, *NVCC_FLAGS, *extra, "-o", str(LIB), *[str(CSRC / s) for s in SOURCES]]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
