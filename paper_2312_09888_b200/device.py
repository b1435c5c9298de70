"""Device / pinned-host memory handles for the ctypes layer.

The product path is plain ctypes over libnekb200 (no torch dependency);
torch tensors, CuPy arrays or anything exposing ``__cuda_array_interface__``
are accepted wherever a device array is expected, and are BORROWED (the
zero-copy contract of include/nekb200.h -- a deliberate divergence from the
reference's copying FieldArray, data_model.py:41-44, because the north star
requires reading "straight from device-resident fields").
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N


def device_ptr(obj) -> int:
    """Raw device address of a borrowed device array (0 for None)."""
    if obj is None:
        return 0
    if isinstance(obj, DeviceArray):
        return obj.ptr
    if isinstance(obj, int):
        return obj
    cai = getattr(obj, "__cuda_array_interface__", None)
    if cai is not None:
        return int(cai["data"][0])
    dp = getattr(obj, "data_ptr", None)
    if dp is not None and getattr(obj, "is_cuda", False):
        return int(dp())
    raise TypeError(f"not a device array: {type(obj).__name__}")


def is_device_array(obj) -> bool:
    if isinstance(obj, DeviceArray):
        return True
    if hasattr(obj, "__cuda_array_interface__"):
        return True
    return bool(getattr(obj, "is_cuda", False))


class DeviceArray:
    """A device allocation owned by libnekb200 (freed on .free() / GC)."""

    def __init__(self, ctx, ptr: int, shape, dtype, owned: bool = True):
        self._ctx = ctx
        self.ptr = int(ptr)
        self.shape = tuple(int(s) for s in np.atleast_1d(shape)) if shape != () else ()
        self.dtype = np.dtype(dtype)
        self._owned = owned

    @property
    def size(self) -> int:
        return int(np.prod(self.shape)) if self.shape else 1

    @property
    def nbytes(self) -> int:
        return self.size * self.dtype.itemsize

    @classmethod
    def empty(cls, ctx, shape, dtype=np.float64) -> "DeviceArray":
        nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
        p = C.c_void_p()
        N.call("nkb_device_alloc", ctx.handle, nbytes, C.byref(p))
        return cls(ctx, p.value or 0, shape, dtype)

    @classmethod
    def from_host(cls, ctx, arr: np.ndarray, stream: int = 0) -> "DeviceArray":
        a = np.ascontiguousarray(arr)
        d = cls.empty(ctx, a.shape, a.dtype)
        d.upload(a, stream)
        return d

    def upload(self, arr: np.ndarray, stream: int = 0, sync: bool = True) -> None:
        a = np.ascontiguousarray(arr)
        if a.nbytes != self.nbytes:
            raise ValueError(f"size mismatch: host {a.nbytes} B vs device {self.nbytes} B")
        N.call("nkb_memcpy", self.ptr, a.ctypes.data, a.nbytes, 1, stream or None)
        if sync:
            N.call("nkb_stream_sync", stream or None)

    def to_host(self, out: np.ndarray | None = None, stream: int = 0) -> np.ndarray:
        if out is None:
            out = np.empty(self.shape, self.dtype)
        N.call("nkb_memcpy", out.ctypes.data, self.ptr, self.nbytes, 2, stream or None)
        N.call("nkb_stream_sync", stream or None)
        return out

    @property
    def __cuda_array_interface__(self):
        return {
            "shape": self.shape,
            "typestr": self.dtype.str,
            "data": (self.ptr, False),
            "version": 3,
            "strides": None,
        }

    def free(self) -> None:
        if self._owned and self.ptr:
            try:
                N.lib().nkb_device_free(self._ctx.handle, self.ptr)
            except Exception:
                pass
        self.ptr = 0

    def __del__(self):
        if getattr(self, "_ctx", None) is not None and self._ctx.handle:
            self.free()


class PinnedBuffer:
    """Page-locked host memory with a numpy view (fast H2D/D2H for e2e)."""

    def __init__(self, nbytes: int):
        p = C.c_void_p()
        N.call("nkb_host_alloc", int(nbytes), C.byref(p))
        self.ptr = p.value or 0
        self.nbytes = int(nbytes)

    def view(self, shape, dtype=np.float64) -> np.ndarray:
        n = int(np.prod(shape)) * np.dtype(dtype).itemsize
        if n > self.nbytes:
            raise ValueError("view larger than the pinned buffer")
        buf = (C.c_byte * n).from_address(self.ptr)
        return np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape)

    def free(self) -> None:
        if self.ptr:
            N.lib().nkb_host_free(self.ptr)
            self.ptr = 0

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass
