"""Build libnekb200.so in-tree with nvcc for sm_100a (no JIT cache: the .so
travels to the GPU box with the repo snapshot).

    python -m paper_2312_09888_b200.build        # or __graft_entry__.build()

Flags that matter for parity: ``-fmad=false`` (no implicit FMA contraction;
every fused multiply-add in the kernels is an explicit fma) and
``-ffp-contract=off`` for host code, matching the CPU oracle's build.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libnekb200.so")
SOURCES = ["abi.cu", "abi_collective.cu", "fused.cu", "stream.cu", "raster.cu", "composite.cu", "mesh_export.cu", "stats.cu", "dssum.cu", "gll.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _flags():
    return ARCH + [
        "-O3", "-lineinfo", "-std=c++17", "-fmad=false",
        "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
        "-I", os.path.join(ROOT, "include"), "-I", CSRC,
    ]


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


CHECKED_LIB = os.path.join(LIBDIR, "libnekb200_checked.so")


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    """Build libnekb200.so; checked=True builds libnekb200_checked.so instead:
    the same sources with -DNKB_CHECKED (device bounds checks, checked.cuh)."""
    os.makedirs(LIBDIR, exist_ok=True)
    objdir = os.path.join(ROOT, "build", "obj_checked" if checked else "obj")
    lib_path = CHECKED_LIB if checked else LIB
    os.makedirs(objdir, exist_ok=True)
    headers = [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".h", ".cuh"))]
    headers.append(os.path.join(ROOT, "include", "nekb200.h"))
    cc = nvcc()
    jobs = []
    objs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(objdir, src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            jobs.append([cc, *_flags(), *(["-DNKB_CHECKED"] if checked else []), "-c", s, "-o", o])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose:
            sys.stderr.write(r.stderr)
        return r

    with ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        list(ex.map(run, jobs))
    if force or jobs or _stale(lib_path, objs):
        run([cc, *ARCH, "-shared", "-o", lib_path, *objs, "-ldl", "-cudart", "static"])
    if checked:
        return lib_path
    # FP64 peak probe (tools/fp64_probe.cu): the bench's FP64 roofline denominator
    probe_src = os.path.join(ROOT, "tools", "fp64_probe.cu")
    probe = os.path.join(LIBDIR, "libnkbprobe.so")
    if os.path.exists(probe_src) and (force or _stale(probe, [probe_src])):
        run([cc, *ARCH, "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", probe_src, "-o", probe,
             "-cudart", "static"])
    # the plain-C usage example (examples/insitu_c_api.c), linked against the library
    ex_src = os.path.join(ROOT, "examples", "insitu_c_api.c")
    ex_bin = os.path.join(LIBDIR, "insitu_c_api")
    if os.path.exists(ex_src) and (force or _stale(ex_bin, [ex_src, LIB, os.path.join(ROOT, "include", "nekb200.h")])):
        run([shutil.which("gcc") or "gcc", "-O2", "-std=c11", "-I", os.path.join(ROOT, "include"), ex_src,
             "-o", ex_bin, "-L", LIBDIR, "-lnekb200", "-Wl,-rpath,$ORIGIN", "-lm"])
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, checked="--checked" in sys.argv))
