"""Build the in-tree CUDA library libboltz_cuda.so for sm_100a.

    python -m paper_1301_4195_b200.build [--verbose]

Explicit nvcc (no JIT, no torch extension cache): the .so lands next to this
file so it travels with the repo snapshot to the GPU box.
"""
from __future__ import annotations

import os
import pathlib
import subprocess
import sys

PKG = pathlib.Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libboltz_cuda.so"
SOURCES = [CSRC / "boltz_cuda.cu", CSRC / "host_weights.cpp", CSRC / "halo.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    return str(pathlib.Path(cuda) / "bin" / "nvcc")


def _inputs():
    return SOURCES + sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + [PKG.parent / "include" / "boltz_cuda.h"]


def up_to_date() -> bool:
    if not LIB.exists():
        return False
    t = LIB.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in _inputs())


def build(verbose: bool = False, force: bool = False, out: pathlib.Path = LIB, defines=()) -> pathlib.Path:
    """Compile libboltz_cuda.so (or a development variant with extra -D defines)."""
    if not force and out == LIB and up_to_date():
        return LIB
    out.parent.mkdir(parents=True, exist_ok=True)
    cmd = [
        _nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "--shared", "-Xcompiler", "-fPIC,-fopenmp",
        "-ccbin", "/usr/bin/g++", *[f"-D{d}" for d in defines], "-o", str(out), *map(str, SOURCES), "-lgomp", "-ldl",
    ]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    print("[build]", " ".join(cmd), file=sys.stderr, flush=True)  # stdout belongs to callers (bench.py's JSON)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or r.returncode != 0:
        sys.stdout.write(r.stdout)
        sys.stderr.write(r.stderr)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed building libboltz_cuda.so")
    return LIB


if __name__ == "__main__":
    build(verbose="--verbose" in sys.argv, force=True)
