"""The maintainer-side stub of INTEGRATION.md §1, as a file: a `gpu_render`
sink kind for the reference (`nekmini`) that renders through libnekb200's C
ABI (`nkb_render_structured`), and `register()`, which adds the kind to the
reference's three closed registries -- `KINDS` and `_KNOWN_ATTRS`
(nekmini/bridge.py:32-39) and `_SINK_TYPES` (nekmini/sinks.py:405-410).

Only ctypes and numpy: nothing from this repository's Python package, so it
is exactly what a reference maintainer would drop next to sinks.py.
tests/test_integration_stub.py runs it against the reference's own Bridge.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

LIB = os.environ.get("NKB_LIB", os.path.join(os.path.dirname(os.path.abspath(__file__)), os.pardir,
                                             "paper_2312_09888_b200", "lib", "libnekb200.so"))
_L = None


def _lib():
    global _L
    if _L is None:
        _L = C.CDLL(LIB)
        _L.nkb_last_error.restype = C.c_char_p
    return _L


def _ok(rc):
    if rc == 0:
        return
    msg = _lib().nkb_last_error().decode()
    # status -> the reference's exception vocabulary (nekb200.h)
    raise (ValueError if rc in (1, 2) else OSError if rc == 3 else RuntimeError)(msg)


class GpuRenderSink:
    """Same contract as the reference's RenderSink (sinks.py:327-351)."""

    def __init__(self, params):
        from nekmini.sinks import _probe_writable

        self.dir = Path(params.get("dir", "render_out"))
        self.dir.mkdir(parents=True, exist_ok=True)
        _probe_writable(self.dir)
        self.w, self.h = int(params.get("width", 256)), int(params.get("height", 256))
        f = params.get("field")
        self.fields = [f] if f else ["temperature", "velocity:mag"]
        self.vmin = float(params["vmin"]) if "vmin" in params else float("nan")
        self.vmax = float(params["vmax"]) if "vmax" in params else float("nan")
        self.ctx = None                       # created on first consume (needs the GPU)

    def consume(self, s) -> int:
        from nekmini.sinks import ImageRGB, write_ppm

        L = _lib()
        if self.ctx is None:
            ctx = C.c_void_p()
            _ok(L.nkb_ctx_create(0, C.byref(ctx)))
            self.ctx = ctx
        total = 0
        for name in self.fields:
            base, _, der = name.partition(":")
            blocks = s.blocks                 # tiled along x in producer order (assemble_global)
            comps = blocks[0].field_named(base).components
            dptr = []
            try:
                for b in blocks:              # H2D: the reference keeps its fields on the host
                    v = np.ascontiguousarray(b.field_named(base).values, dtype=np.float64)
                    p = C.c_void_p()
                    _ok(L.nkb_device_alloc(self.ctx, C.c_int64(v.nbytes), C.byref(p)))
                    dptr.append(p)
                    _ok(L.nkb_memcpy(p, C.c_void_p(v.ctypes.data), C.c_int64(v.nbytes), 1, None))
                ni = (C.c_int64 * len(blocks))(*[b.dims[0] for b in blocks])
                ptrs = (C.c_void_p * len(blocks))(*[p.value for p in dptr])
                rgb = C.c_void_p()
                _ok(L.nkb_device_alloc(self.ctx, C.c_int64(3 * self.w * self.h), C.byref(rgb)))
                dptr.append(rgb)
                _, nj, nk = blocks[0].dims
                _ok(L.nkb_render_structured(self.ctx, len(blocks), ptrs, ni, C.c_int64(nj * nk), comps,
                                            1 if der == "mag" else 0, self.w, self.h, C.c_double(self.vmin),
                                            C.c_double(self.vmax), rgb, None, None))
                out = np.empty(3 * self.w * self.h, np.uint8)
                _ok(L.nkb_memcpy(C.c_void_p(out.ctypes.data), rgb, C.c_int64(out.nbytes), 2, None))
                _ok(L.nkb_stream_sync(None))
            finally:
                for p in dptr:
                    L.nkb_device_free(self.ctx, p)
            total += write_ppm(ImageRGB(self.w, self.h, out.tobytes()),
                               self.dir / f"step{s.step:06d}_{name.replace(':', '_')}.ppm")
        return total

    def finalize(self):
        if self.ctx is not None:
            _lib().nkb_ctx_destroy(self.ctx)
            self.ctx = None


def register(kind: str = "gpu_render"):
    """Add `kind` to nekmini's closed registries (bridge.py:32-39, sinks.py:405-410)."""
    from nekmini import bridge, sinks

    if kind not in bridge.KINDS:
        bridge.KINDS = tuple(bridge.KINDS) + (kind,)
    bridge._KNOWN_ATTRS[kind] = set(bridge._KNOWN_ATTRS["render"])
    sinks._SINK_TYPES[kind] = GpuRenderSink
    return kind
