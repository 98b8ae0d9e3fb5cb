"""The C++ view of the boundary (include/boltz_cuda.hpp) compiles against the
library on CPU and runs on a GPU."""
import pathlib
import subprocess

import pytest

from paper_1301_4195_b200.build import LIB, build

REPO = pathlib.Path(__file__).resolve().parent.parent
EXE = REPO / "tests" / "cpp" / "wrapper_demo"


def _compile():
    build()
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", str(REPO / "include"), "-o", str(EXE),
                    str(REPO / "tests" / "cpp" / "wrapper_demo.cpp"), str(LIB), f"-Wl,-rpath,{LIB.parent}"],
                   check=True)


def test_cpp_wrapper_compiles():
    _compile()
    assert EXE.exists()


@pytest.mark.gpu
def test_cpp_wrapper_runs(gpu):
    _compile()
    out = subprocess.run([str(EXE)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "collide ok" in out.stdout and "config error category 2" in out.stdout
    ratio = float(out.stdout.split("=")[1].split()[0])
    assert ratio < 1e-12
