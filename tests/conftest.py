import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests", "golden")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C ABI)")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the native library and the oracle once (no-op when up to date)."""
    from oracle import oracle as orc
    from paper_2312_09888_b200 import build as nb

    nb.build()
    orc.build()


@pytest.fixture(scope="session")
def ctx():
    from paper_2312_09888_b200.context import Context

    c = Context(0)
    yield c
    c.close()


@pytest.fixture(params=["geo_cached", "geo_uncached"])
def ctx_geo(request, ctx):
    """The session context with the per-mesh geometry cache on or off: both
    fused-kernel variants must give bit-identical results."""
    on = request.param == "geo_cached"
    ctx.set_geometry_cache(on)
    yield ctx
    ctx.set_geometry_cache(True)
