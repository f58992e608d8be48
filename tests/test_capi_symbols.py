"""The drop-in boundary: libgnw.so loads, exports every entry point include/gnw.h declares,
links no oracle code, and fails loudly (no CPU fallback) without a GPU."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_2209_02815_b200 import _capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "gnw.h")).read()
    return sorted(set(re.findall(r"\b(gnw_[a-z_]+)\s*\(", src)))


def test_header_and_binding_agree():
    assert declared() == sorted(_capi.EXPORTED)


def test_every_symbol_exported():
    lib = _capi.load()
    for name in declared():
        assert hasattr(lib, name), name


def test_no_oracle_or_reference_code_linked():
    out = subprocess.run(["nm", "-D", "--defined-only", _capi.LIB_PATH], capture_output=True, text=True).stdout
    assert "orc_" not in out
    assert "ertinv" not in out
    assert "gnw_minres_solve" in out


def test_sm100a_only_cubin():
    out = subprocess.run(["cuobjdump", "--list-elf", _capi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert re.search(r"sm_(?!100a)\d+", out.replace("sm_100a", "")) is None


def test_dmma_present_in_sass():
    sass = subprocess.run(["cuobjdump", "-sass", _capi.LIB_PATH], capture_output=True, text=True).stdout
    assert "DMMA" in sass  # FP64 tensor-core capacitance GEMM


def test_version_and_create_without_gpu():
    lib = _capi.load()
    assert b"sm_100a" in lib.gnw_version()
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    h = ctypes.c_void_p()
    dev = (ctypes.c_int * 1)(0)
    rc = lib.gnw_create(1, dev, ctypes.byref(h))
    assert rc == _capi.GNW_DEVICE
    assert b"no CUDA device" in lib.gnw_last_error()
