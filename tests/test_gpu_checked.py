"""The device bounds-checked build (libnekb200_checked.so, -DNKB_CHECKED:
checked.cuh).  compute-sanitizer is closed on the GPU pool, so the hot
kernels check their own shared- and global-memory indices; this runs a
workload that launches every hot-path kernel (tools/sanitize_case.py) on the
checked library and requires zero violations, and proves a violation does
surface (NKB_CHECKED_SELFTEST=1 plants one failing check)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_2312_09888_b200", "lib", "libnekb200_checked.so")


def _run(extra_env):
    env = dict(os.environ, NKB_LIB=CHECKED, **extra_env)
    return subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_case.py")], env=env,
                          capture_output=True, text=True, timeout=600)


@pytest.mark.skipif(not os.path.exists(CHECKED), reason="checked build missing (build(checked=True))")
def test_every_hot_kernel_passes_its_bounds_checks():
    r = _run({})
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "sanitize case done" in r.stdout


@pytest.mark.skipif(not os.path.exists(CHECKED), reason="checked build missing (build(checked=True))")
def test_a_failed_check_surfaces_as_an_error():
    r = _run({"NKB_CHECKED_SELFTEST": "1"})
    assert r.returncode != 0
    assert "device bounds check failed" in (r.stdout + r.stderr)
