import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libgnw.so's CUDA kernels)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def oracles():
    """The plain-C restatement, plus the compiled reference when available."""
    import orc

    out = {}
    if not orc.available("restatement"):
        orc.build("restatement")
    out["restatement"] = orc.Oracle("restatement")
    if not orc.available("reference") and os.path.isdir("/root/reference/proj/src"):
        orc.build("reference")
    if orc.available("reference"):
        out["reference"] = orc.Oracle("reference")
    return out


@pytest.fixture(scope="session")
def oracle(oracles):
    """Prefer the unmodified reference; the restatement is pinned bit-exact to it."""
    return oracles.get("reference", oracles["restatement"])


@pytest.fixture(scope="session")
def gpu_ctx_factory():
    from paper_2209_02815_b200 import Context

    def make(mesh, opts=None, exact=False):
        c = Context(0)
        c.set_coarse_mode(exact)
        c.assemble(mesh, opts)
        return c

    return make
