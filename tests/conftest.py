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


@pytest.fixture(params=["geo_compact", "geo_full", "geo_uncached"])
def ctx_geo(request, ctx):
    """The session context with the per-mesh geometry cache in its default
    (compact when every element is extruded) or full layout, or off: every
    fused-kernel variant must give bit-identical results."""
    ctx.set_geometry_cache({"geo_compact": "auto", "geo_full": "full", "geo_uncached": False}[request.param])
    yield ctx
    ctx.set_geometry_cache(True)
