"""The C++ drop-in face (include/gnw.hpp) compiles against the reference-style caller,
links libgnw.so, and (on a GPU) reproduces the reference's Woodbury-vs-Laplace test."""
import os
import subprocess

import pytest

from paper_2209_02815_b200 import _capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "gn_step_example.cpp")
BIN = os.path.join(ROOT, "tests", "cpp", "gn_step_example")


def build():
    libdir = os.path.dirname(_capi.LIB_PATH)
    subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", f"-I{ROOT}/include", SRC, "-o", BIN,
                    f"-L{libdir}", "-lgnw", f"-Wl,-rpath,{libdir}"], check=True)


def test_cpp_caller_compiles_and_links():
    _capi.load()
    build()
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_cpp_caller_runs_on_gpu():
    build()
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "woodbury" in out.stdout
