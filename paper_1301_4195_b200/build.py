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


REF_INCLUDE = pathlib.Path("/root/reference/proj/include")
REF_GRID_SRC = pathlib.Path("/root/reference/proj/src/velocity_grid.cpp")
SHIM_DEMO = PKG.parent / "tests" / "cpp" / "ref_shim_demo"


def build_shim(force: bool = False):
    """Compile the reference-typed drop-in (shim/fourier_cuda.cpp implementing
    the reference's unmodified boltz::SpectralTransform, shim/collision_cuda.cpp)
    together with the reference's own velocity_grid.cpp, compiled in place,
    into tests/cpp/ref_shim_demo.  Needs the reference tree (this container);
    the GPU box runs the prebuilt binary.  Returns the binary or None."""
    if not (REF_INCLUDE.is_dir() and REF_GRID_SRC.is_file()):
        return SHIM_DEMO if SHIM_DEMO.exists() else None
    lib = build()
    srcs = [PKG.parent / "tests" / "cpp" / "ref_shim_demo.cpp", PKG / "shim" / "fourier_cuda.cpp",
            PKG / "shim" / "collision_cuda.cpp", REF_GRID_SRC]
    deps = srcs + [lib, PKG.parent / "include" / "boltz_cuda.hpp", PKG / "shim" / "collision_cuda.hpp"]
    if not force and SHIM_DEMO.exists() and all(p.stat().st_mtime <= SHIM_DEMO.stat().st_mtime for p in deps):
        return SHIM_DEMO
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-I", str(REF_INCLUDE), "-I", str(PKG.parent / "include"),
           "-I", str(PKG / "shim"), "-o", str(SHIM_DEMO), *map(str, srcs), str(lib),
           f"-Wl,-rpath,{lib.parent}"]
    print("[build]", " ".join(cmd), file=sys.stderr, flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("g++ failed building tests/cpp/ref_shim_demo")
    return SHIM_DEMO


if __name__ == "__main__":
    build(verbose="--verbose" in sys.argv, force=True)
