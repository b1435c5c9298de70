"""Thin object wrapper over one libnekb200 context (one per process and GPU,
confined to one host thread -- reference bridge.py:132-137)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .device import DeviceArray, device_ptr


@dataclass(frozen=True)
class Report:
    """Per-execute report (the SinkReport payload of the in situ analysis)."""

    n_triangles: int
    n_triangles_global: int
    tri_capacity: int
    range: tuple[float, float]
    data_range: tuple[float, float]
    ms_fused: float
    ms_raster: float
    ms_composite: float
    ms_resolve: float
    reran: bool
    geometry_cached: bool = False
    ms_geometry: float = 0.0
    surface_pass: int = 0          # 0: K1 fused, 1: K1s stream (no gradient), 2: K1g (cached geometry)
    overflowed: bool = False       # execute_async steps only: triangles overflowed (result incomplete)
    composite_overlapped: bool = False   # execute_async P2P steps: composite beside the next surface pass

    @classmethod
    def from_native(cls, r: N.NkbReport) -> "Report":
        return cls(
            int(r.n_triangles), int(r.n_triangles_global), int(r.tri_capacity),
            (float(r.range[0]), float(r.range[1])),
            (float(r.data_range[0]), float(r.data_range[1])),
            float(r.ms_fused), float(r.ms_raster), float(r.ms_composite), float(r.ms_resolve),
            bool(r.reran), bool(r.geometry_cached), float(r.ms_geometry), int(r.surface_pass),
            bool(r.overflowed), bool(r.composite_overlapped),
        )


def gll(order: int = 7) -> tuple[np.ndarray, np.ndarray]:
    """GLL nodes and differentiation matrix exactly as the kernels use them."""
    x = np.zeros(order + 1)
    D = np.zeros((order + 1, order + 1))
    N.call("nkb_gll", order, x.ctypes.data, D.ctypes.data)
    return x, D


def device_count() -> int:
    n = C.c_int(0)
    rc = N.lib().nkb_device_count(C.byref(n))
    return int(n.value) if rc == N.NKB_OK else 0


class Context:
    def __init__(self, device: int = 0):
        h = C.c_void_p()
        N.call("nkb_ctx_create", int(device), C.byref(h))
        self.handle = h.value
        self.device = int(device)
        self.rank = 0
        self.nranks = 1

    # -- lifetime --------------------------------------------------------------
    def close(self) -> None:
        if self.handle:
            self._wait_ppm_readers()            # an async PPM write may still read pinned memory
            N.lib().nkb_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- DataAdaptor ------------------------------------------------------------
    def mesh_set(self, n_elements: int, x, y, z, order: int = 7, element_offset: int = 0,
                 n_elements_global: int = 0) -> None:
        N.call("nkb_mesh_set", self.handle, int(n_elements), int(order), device_ptr(x), device_ptr(y),
               device_ptr(z), int(element_offset), int(n_elements_global))

    def mesh_set_global_ids(self, gid, stream: int = 0) -> None:
        """Global node ids (device int64, one per GLL copy): builds the DSSUM
        gather-scatter (collective with a communicator)."""
        N.call("nkb_mesh_set_global_ids", self.handle, device_ptr(gid), stream or None)

    def dssum(self, field, stream: int = 0) -> None:
        """In-place direct stiffness average of a device point field."""
        N.call("nkb_dssum", self.handle, device_ptr(field), stream or None)

    def transit_gather(self, root: int = 0, stream: int = 0) -> None:
        """N:1 GPU-direct staging: gather every rank's mesh + fields to `root`
        (collective); root's context then holds the assembled mesh."""
        N.call("nkb_transit_gather", self.handle, int(root), stream or None)

    def mesh_modified(self) -> None:
        """Coordinates were edited in place (moving mesh): drop the geometry cache."""
        N.call("nkb_mesh_modified", self.handle)

    def set_geometry_cache(self, enable: bool | str) -> None:
        """True / "auto": cache (compact layout when every element is extruded);
        "full": cache in the full 72 B/point layout; False: recompute every step."""
        mode = {"auto": 1, "full": 2}.get(enable, None) if isinstance(enable, str) else int(bool(enable))
        if mode is None:
            raise ValueError(f"geometry cache mode must be True, False, 'auto' or 'full', got {enable!r}")
        N.call("nkb_set_geometry_cache", self.handle, mode)

    def geometry_info(self) -> dict:
        """{"layout": "none" | "full" | "compact", "bytes": device bytes of the cache}."""
        lay, nb = C.c_int(0), C.c_int64(0)
        N.call("nkb_geometry_info", self.handle, C.byref(lay), C.byref(nb))
        return {"layout": ("none", "full", "compact")[lay.value], "bytes": int(nb.value)}

    def field_set(self, name: str, base, ncomp: int = 1, comp_stride: int = 0) -> None:
        N.call("nkb_field_set", self.handle, name.encode(), int(ncomp), device_ptr(base), int(comp_stride))

    def field_clear(self) -> None:
        N.call("nkb_field_clear", self.handle)

    def set_velocity_name(self, name: str) -> None:
        N.call("nkb_set_velocity_name", self.handle, name.encode())

    def metadata(self) -> N.NkbMeshMetadata:
        m = N.NkbMeshMetadata()
        N.call("nkb_get_mesh_metadata", self.handle, C.byref(m))
        return m

    def bounds(self, stream: int = 0) -> tuple[float, ...]:
        out = np.zeros(6)
        N.call("nkb_mesh_bounds", self.handle, out.ctypes.data, stream or None)
        return tuple(float(v) for v in out)

    def get_mesh(self, points=None, conn=None, offsets=None, types=None, stream: int = 0) -> None:
        N.call("nkb_get_mesh", self.handle, device_ptr(points), device_ptr(conn), device_ptr(offsets),
               device_ptr(types), stream or None)

    def array_components(self, name: str) -> int:
        n = C.c_int(0)
        N.call("nkb_array_components", self.handle, name.encode(), C.byref(n))
        return int(n.value)

    def add_array(self, name: str, out, association: int = N.NKB_ASSOC_POINT, stream: int = 0) -> int:
        n = C.c_int(0)
        N.call("nkb_add_array", self.handle, name.encode(), int(association), device_ptr(out), C.byref(n),
               stream or None)
        return int(n.value)

    # -- AnalysisAdaptor::Execute ---------------------------------------------------
    def execute(self, pipeline: N.NkbPipeline, stream: int = 0) -> Report:
        r = N.NkbReport()
        N.call("nkb_execute", self.handle, C.byref(pipeline), C.byref(r), stream or None)
        return Report.from_native(r)

    def execute_async(self, pipeline: N.NkbPipeline, stream: int = 0) -> None:
        """Enqueue one step without a host synchronisation (nkb_execute_async)."""
        N.call("nkb_execute_async", self.handle, C.byref(pipeline), stream or None)

    def wait(self, stream: int = 0) -> Report:
        """Synchronise and return the report of the last execute_async step."""
        r = N.NkbReport()
        N.call("nkb_execute_wait", self.handle, C.byref(r), stream or None)
        return Report.from_native(r)

    def image(self, width: int, height: int, depth: bool = False, stream: int = 0):
        rgba = np.empty((height, width, 4), np.uint8)
        dep = np.empty((height, width), np.float32) if depth else None
        N.call("nkb_image_copy", self.handle, rgba.ctypes.data, dep.ctypes.data if depth else None,
               stream or None)
        return (rgba, dep) if depth else rgba

    def hold_ppm(self, future) -> None:
        """Register a pending reader of the pinned PPM buffer (an asynchronous
        file write); image_ppm() and close() wait for it before the buffer is
        overwritten or freed."""
        self._ppm_readers = [f for f in getattr(self, "_ppm_readers", []) if not f.done()] + [future]

    def _wait_ppm_readers(self) -> None:
        readers, self._ppm_readers = getattr(self, "_ppm_readers", []), []
        for f in readers:
            f.exception()           # wait; the owning sink re-raises its own error

    def image_ppm(self, stream: int = 0) -> memoryview:
        """The last image as complete PPM bytes (header + RGB), packed on the
        GPU into library-owned pinned memory; valid until the next call (which
        first waits for every registered reader of the previous bytes)."""
        self._wait_ppm_readers()
        ptr, n = C.c_void_p(), C.c_int64()
        N.call("nkb_image_ppm", self.handle, C.byref(ptr), C.byref(n), stream or None)
        return memoryview((C.c_ubyte * n.value).from_address(ptr.value)).cast("B")

    def stats(self, segments, collective: bool = False, stream: int = 0) -> tuple[float, float, float]:
        """(min, max, mean) of the concatenated device segments
        [(ptr, n_tuples, ncomp, comp_stride), ...] in AoS order, with numpy's
        arithmetic (nkb_stats); collective: over all ranks in rank order."""
        arr = (N.NkbSegment * max(1, len(segments)))()
        for i, (ptr, n, nc, st) in enumerate(segments):
            arr[i] = N.NkbSegment(C.c_void_p(int(ptr)), int(n), int(nc), int(st))
        out = (C.c_double * 3)()
        N.call("nkb_stats", self.handle, arr, len(segments), int(bool(collective)), out, stream or None)
        return float(out[0]), float(out[1]), float(out[2])

    def composite_partitions(self, parts, pipeline: N.NkbPipeline, stream: int = 0) -> None:
        """Depth-composite the key buffers of partition contexts on this
        device into this context's image (nkb_composite_partitions)."""
        arr = (C.c_void_p * len(parts))(*[c.handle for c in parts])
        N.call("nkb_composite_partitions", self.handle, arr, len(parts), C.byref(pipeline), stream or None)

    def image_device(self) -> tuple[int, int, int]:
        a, b, c = C.c_void_p(), C.c_void_p(), C.c_void_p()
        N.call("nkb_image_device", self.handle, C.byref(a), C.byref(b), C.byref(c))
        return a.value or 0, b.value or 0, c.value or 0

    def triangles(self, with_meta: bool = False):
        """Triangles of the last execute, copied to host: (n, 3, 4) float32 [+ meta uint64]."""
        t, m, n = C.c_void_p(), C.c_void_p(), C.c_int64()
        N.call("nkb_triangles_device", self.handle, C.byref(t), C.byref(m), C.byref(n))
        cnt = int(n.value)
        tri = np.empty((cnt, 3, 4), np.float32)
        if cnt:
            N.call("nkb_memcpy", tri.ctypes.data, t.value, tri.nbytes, 2, None)
        meta = None
        if with_meta:
            meta = np.empty(cnt, np.uint64)
            if cnt and m.value:
                N.call("nkb_memcpy", meta.ctypes.data, m.value, meta.nbytes, 2, None)
        N.call("nkb_stream_sync", None)
        return (tri, meta) if with_meta else tri

    # -- composite communicator ----------------------------------------------------
    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (C.c_ubyte * 128)()
        N.call("nkb_nccl_unique_id", C.addressof(buf))
        return bytes(buf)

    def comm_init(self, uid: bytes, nranks: int, rank: int) -> None:
        buf = (C.c_ubyte * 128).from_buffer_copy(uid)
        N.call("nkb_comm_init", self.handle, C.addressof(buf), int(nranks), int(rank))
        self.rank, self.nranks = int(rank), int(nranks)

    def comm_destroy(self) -> None:
        N.call("nkb_comm_destroy", self.handle)
        self.rank, self.nranks = 0, 1

    # -- reference 2D renderer -------------------------------------------------------
    def render_structured(self, blocks, rows: int, comps: int, mode: int, width: int, height: int,
                          vmin: float, vmax: float, rgb_out, stream: int = 0) -> tuple[float, float]:
        nb = len(blocks)
        ptrs = (C.c_void_p * nb)(*[device_ptr(v) for v, _ in blocks])
        nis = (C.c_int64 * nb)(*[int(ni) for _, ni in blocks])
        rng = np.zeros(2)
        N.call("nkb_render_structured", self.handle, nb, C.addressof(ptrs), C.addressof(nis), int(rows),
               int(comps), int(mode), int(width), int(height), float(vmin), float(vmax), device_ptr(rgb_out),
               rng.ctypes.data, stream or None)
        return float(rng[0]), float(rng[1])

    def alloc(self, shape, dtype=np.float64) -> DeviceArray:
        return DeviceArray.empty(self, shape, dtype)

    def upload(self, arr: np.ndarray, stream: int = 0) -> DeviceArray:
        return DeviceArray.from_host(self, arr, stream)
