"""ctypes binding of libnekb200.so (include/nekb200.h).

The product path has no fallback: if the shared library is missing or the
CUDA runtime fails, calls raise.  Status codes map onto the reference's
exception vocabulary: EINVAL/ERANGE -> ValueError,
EIO -> OSError, ECUDA/ENCCL/ESTATE -> RuntimeError, so `Bridge.update`'s
sink isolation (reference bridge.py:164-176) catches them unchanged.
"""
from __future__ import annotations

import ctypes as C
import math
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libnekb200.so")

NKB_OK, NKB_EINVAL, NKB_ERANGE, NKB_EIO, NKB_ECUDA, NKB_ENCCL, NKB_ESTATE = range(7)
NKB_SURF_ISO, NKB_SURF_SLICE = 0, 1
NKB_ASSOC_POINT, NKB_ASSOC_CELL = 0, 1
NKB_VTK_HEXAHEDRON = 12
NKB_MAX_SURFACES = 4
NKB_MAX_ANCHORS = 8
NKB_NAME_MAX = 64


class NativeError(RuntimeError):
    """CUDA / NCCL / call-order failure inside libnekb200."""


class NkbSurface(C.Structure):
    _fields_ = [
        ("kind", C.c_int),
        ("field", C.c_char * NKB_NAME_MAX),
        ("value", C.c_double),
        ("normal", C.c_double * 3),
    ]


class NkbPipeline(C.Structure):
    _fields_ = [
        ("n_surfaces", C.c_int),
        ("surfaces", NkbSurface * NKB_MAX_SURFACES),
        ("color_field", C.c_char * NKB_NAME_MAX),
        ("width", C.c_int),
        ("height", C.c_int),
        ("view", C.c_double * 12),
        ("vmin", C.c_double),
        ("vmax", C.c_double),
        ("n_anchors", C.c_int),
        ("anchor_t", C.c_double * NKB_MAX_ANCHORS),
        ("anchor_rgb", (C.c_ubyte * 3) * NKB_MAX_ANCHORS),
        ("background", C.c_ubyte * 4),
        ("emit_meta", C.c_int),
        ("composite", C.c_int),
        ("timing", C.c_int),
        ("continuous", C.c_int),
        ("persp", C.c_double * 4),
    ]


class NkbReport(C.Structure):
    _fields_ = [
        ("n_triangles", C.c_int64),
        ("n_triangles_global", C.c_int64),
        ("tri_capacity", C.c_int64),
        ("range", C.c_double * 2),
        ("data_range", C.c_double * 2),
        ("ms_fused", C.c_float),
        ("ms_raster", C.c_float),
        ("ms_composite", C.c_float),
        ("ms_resolve", C.c_float),
        ("reran", C.c_int),
        ("geometry_cached", C.c_int),
        ("ms_geometry", C.c_float),
        ("surface_pass", C.c_int),
        ("overflowed", C.c_int),
        ("composite_overlapped", C.c_int),
    ]


class NkbSegment(C.Structure):
    _fields_ = [
        ("base", C.c_void_p),
        ("n_tuples", C.c_int64),
        ("ncomp", C.c_int),
        ("comp_stride", C.c_int64),
    ]


class NkbMeshMetadata(C.Structure):
    _fields_ = [
        ("n_elements", C.c_int64),
        ("order", C.c_int),
        ("n_points", C.c_int64),
        ("n_cells", C.c_int64),
        ("cell_type", C.c_int),
        ("element_offset", C.c_int64),
        ("n_elements_global", C.c_int64),
        ("n_fields", C.c_int),
        ("rank", C.c_int),
        ("nranks", C.c_int),
    ]


_vp = C.c_void_p
_i64 = C.c_int64
_SIGS = {
    "nkb_abi_version": ([], C.c_int),
    "nkb_last_error": ([], C.c_char_p),
    "nkb_ctx_create": ([C.c_int, C.POINTER(_vp)], C.c_int),
    "nkb_ctx_destroy": ([_vp], C.c_int),
    "nkb_gll": ([C.c_int, _vp, _vp], C.c_int),
    "nkb_mesh_set": ([_vp, _i64, C.c_int, _vp, _vp, _vp, _i64, _i64], C.c_int),
    "nkb_field_set": ([_vp, C.c_char_p, C.c_int, _vp, _i64], C.c_int),
    "nkb_field_clear": ([_vp], C.c_int),
    "nkb_get_mesh_metadata": ([_vp, C.POINTER(NkbMeshMetadata)], C.c_int),
    "nkb_mesh_bounds": ([_vp, _vp, _vp], C.c_int),
    "nkb_get_mesh": ([_vp, _vp, _vp, _vp, _vp, _vp], C.c_int),
    "nkb_add_array": ([_vp, C.c_char_p, C.c_int, _vp, C.POINTER(C.c_int), _vp], C.c_int),
    "nkb_array_components": ([_vp, C.c_char_p, C.POINTER(C.c_int)], C.c_int),
    "nkb_set_velocity_name": ([_vp, C.c_char_p], C.c_int),
    "nkb_mesh_modified": ([_vp], C.c_int),
    "nkb_set_geometry_cache": ([_vp, C.c_int], C.c_int),
    "nkb_geometry_info": ([_vp, _vp, _vp], C.c_int),
    "nkb_composite_partitions": ([_vp, _vp, C.c_int, _vp, _vp], C.c_int),
    "nkb_execute_async": ([_vp, _vp, _vp], C.c_int),
    "nkb_execute_wait": ([_vp, _vp, _vp], C.c_int),
    "nkb_execute": ([_vp, C.POINTER(NkbPipeline), C.POINTER(NkbReport), _vp], C.c_int),
    "nkb_image_device": ([_vp, C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_vp)], C.c_int),
    "nkb_image_copy": ([_vp, _vp, _vp, _vp], C.c_int),
    "nkb_image_ppm": ([_vp, C.POINTER(C.c_void_p), C.POINTER(C.c_int64), _vp], C.c_int),
    "nkb_stats": ([_vp, C.POINTER(NkbSegment), C.c_int, C.c_int, C.POINTER(C.c_double), _vp], C.c_int),
    "nkb_encode_be": ([_vp, C.c_char_p, _vp, _i64, C.POINTER(C.c_int64), _vp], C.c_int),
    "nkb_mesh_set_global_ids": ([_vp, _vp, _vp], C.c_int),
    "nkb_dssum": ([_vp, _vp, _vp], C.c_int),
    "nkb_transit_gather": ([_vp, C.c_int, _vp], C.c_int),
    "nkb_triangles_device": ([_vp, C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_i64)], C.c_int),
    "nkb_nccl_unique_id": ([_vp], C.c_int),
    "nkb_comm_init": ([_vp, _vp, C.c_int, C.c_int], C.c_int),
    "nkb_comm_destroy": ([_vp], C.c_int),
    "nkb_render_structured": (
        [_vp, C.c_int, _vp, _vp, _i64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
         _vp, _vp, _vp],
        C.c_int,
    ),
    "nkb_device_alloc": ([_vp, _i64, C.POINTER(_vp)], C.c_int),
    "nkb_device_free": ([_vp, _vp], C.c_int),
    "nkb_host_alloc": ([_i64, C.POINTER(_vp)], C.c_int),
    "nkb_host_free": ([_vp], C.c_int),
    "nkb_memcpy": ([_vp, _vp, _i64, C.c_int, _vp], C.c_int),
    "nkb_stream_sync": ([_vp], C.c_int),
    "nkb_device_sync": ([], C.c_int),
    "nkb_device_count": ([C.POINTER(C.c_int)], C.c_int),
}
EXPORTED = tuple(_SIGS)

_lib = None


def lib():
    """Load libnekb200.so (raises if it was not built -- there is no CPU fallback)."""
    global _lib
    if _lib is None:
        path = os.environ.get("NKB_LIB", LIB_PATH)       # A/B of two builds of the same ABI
        if not os.path.exists(path):
            raise NativeError(
                f"{path} is missing; build it with `python -m paper_2312_09888_b200.build` "
                "(the GPU path has no CPU fallback)"
            )
        L = C.CDLL(path, mode=C.RTLD_GLOBAL)
        for name, (argtypes, restype) in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = argtypes
            fn.restype = restype
        if L.nkb_abi_version() != 1:
            raise NativeError("libnekb200 ABI version mismatch")
        _lib = L
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc == NKB_OK:
        return
    msg = (lib().nkb_last_error() or b"").decode("utf-8", "replace")
    if what:
        msg = f"{what}: {msg}"
    if rc in (NKB_EINVAL, NKB_ERANGE):
        raise ValueError(msg)
    if rc == NKB_EIO:
        raise OSError(msg)
    raise NativeError(msg)


def call(name: str, *args):
    check(getattr(lib(), name)(*args), name)


NAN = math.nan
