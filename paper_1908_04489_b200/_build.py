"""Compile the CUDA library (csrc/ucp_kernels.cu -> libucp_b200.so) for sm_100a.

In-tree build so the .so travels with the repo snapshot to the GPU box.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libucp_b200.so"
SOURCES = [CSRC / "ucp_kernels.cu"]
# every file ucp_kernels.cu includes: an edit to any of them rebuilds the library
HEADERS = sorted(CSRC.glob("*.h")) + sorted(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "ucp_b200.h"]
# stress build (tests/test_gpu_stress.py): schedule jitter + device index checks
STRESS_LIB = PKG / "libucp_b200_stress.so"

NVCC_FLAGS = [
    "-O3",
    "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "-fmad=false",            # ref-order: no FMA contraction in device code
    "-Xcompiler", "-fPIC,-ffp-contract=off",
    "-shared",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def stale(lib: Path = LIB) -> bool:
    if not lib.exists():
        return True
    t = lib.stat().st_mtime
    return any(p.stat().st_mtime > t for p in SOURCES + HEADERS + [Path(__file__)])


def build(force: bool = False, verbose: bool = False, lib: Path = LIB, defines: tuple = ()) -> Path:
    """nvcc the library to ``lib`` (``defines``: extra -D macros for variant builds)."""
    if not force and not stale(lib):
        return lib
    cmd = [nvcc(), *NVCC_FLAGS, *(f"-D{x}" for x in defines), *(str(s) for s in SOURCES), "-o", str(lib) + ".tmp"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({' '.join(cmd)}):\n{res.stdout}\n{res.stderr}")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(str(lib) + ".tmp", lib)
    return lib


def build_stress(force: bool = False) -> Path:
    return build(force=force, lib=STRESS_LIB, defines=("UCP_STRESS",))


if __name__ == "__main__":
    if "--stress" in sys.argv:
        print(build_stress(force="--force" in sys.argv))
    else:
        build(force="--force" in sys.argv, verbose="-v" in sys.argv)
        print(LIB)
