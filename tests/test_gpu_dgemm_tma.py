"""The capacitance GEMM's TMA-staged kernel (dgemm_tma.cu) against the cp.async kernel it replaces
(GNW_DGEMM_TMA=0; the switch is read once per process, so each mode runs in its own process,
tools/check_dgemm_tma.py): the Cholesky factor of C bit for bit, on shapes that exercise the TMA
unit's zero fill -- fewer rows than a 128-row box, a row count just past a tile, and N not a
multiple of the 16-column box."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_tma_dgemm_bitwise_cp_async_on_edge_shapes():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "check_dgemm_tma.py"), "n7m2", "n9m33", "n33m129"],
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert out.stdout.count("bitwise equal: True") == 3, out.stdout[-2000:]
