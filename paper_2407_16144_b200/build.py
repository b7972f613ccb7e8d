"""In-tree build of the product libraries (paper_2407_16144_b200/lib/*.so).

``nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false`` for
the hx CUDA layer, g++ for the host driver and generator (csrc/Makefile).
"""
from __future__ import annotations

import os
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "lib"
GPU_LIB = Path(os.environ["HPLP_GPU_LIB"]) if os.environ.get("HPLP_GPU_LIB") else LIB / "libhplp_gpu.so"
GEN_LIB = LIB / "libhplp_gen.so"


def build(quiet: bool = True, jobs: int = 4) -> None:
    out = subprocess.DEVNULL if quiet else None
    subprocess.run(["make", f"-j{jobs}", "-s"], cwd=CSRC, check=True, stdout=out)


def ensure_built() -> None:
    """Build if the libraries are missing or older than their sources."""
    srcs = [p for p in CSRC.iterdir() if p.suffix in (".cu", ".cuh", ".cpp", ".hpp")]
    srcs += list((PKG.parent / "include").glob("*.h"))
    newest = max(p.stat().st_mtime for p in srcs)
    if os.environ.get("HPLP_GPU_LIB"):
        return
    if not GPU_LIB.exists() or not GEN_LIB.exists() or min(GPU_LIB.stat().st_mtime, GEN_LIB.stat().st_mtime) < newest:
        build()
