"""SEM element blocks on the reference's framed wire (in transit over TCP).

The reference frames every message as (pkg/src/nekmini/wire.py:1-16)::

    magic 'NKSS' | version u8 | tag u8 | payload length u64 LE | payload

and marshals structured blocks as BlockPayload (tag 0x04, :85-124).  SEM
partitions get a new tag, 0x07 (SemBlockPayload), laid out in the same
little-endian style:

    element_offset i64 | n_elements i64 | n_elements_global i64 | order u8
    x, y, z           f64[E*(N+1)^3] each
    field count       u32
    per field         name length u16 + UTF-8 | association u8 (0 point)
                      | components u32 | value count u64 | values f64[] (SoA:
                        component c at [c*npts, (c+1)*npts))

Device-resident arrays are copied straight into the frame buffer (nkb_memcpy
D2H at their offsets), so a producer GPU streams its partition to the socket
without intermediate Python copies.  The GPU-direct alternative,
NCCL send/recv to the endpoint GPU, is nkb_transit_gather (sink kind
``transit``).
"""
from __future__ import annotations

import ctypes
import struct

import numpy as np

from . import _native as N
from .data_model import POINT, FieldArray, SemBlock
from .device import device_ptr, is_device_array

MAGIC = b"NKSS"
VERSION = 0x01
HEADER = struct.Struct("<4sBBQ")
TAG_SEM_BLOCK = 0x07


class ProtocolError(RuntimeError):
    """Malformed or truncated frame (the reference's wire.ProtocolError)."""


def _soa(f: FieldArray, npts: int):
    """(component arrays) of a field in SoA order, host or device."""
    if isinstance(f.values, tuple):
        return list(f.values)
    if is_device_array(f.values):
        stride = f.comp_stride or npts
        base = device_ptr(f.values)
        return [(base + 8 * c * stride, npts) for c in range(f.components)]
    a = np.asarray(f.values, dtype=np.float64)
    if f.components > 1 and not f.comp_stride:
        a = a.reshape(npts, f.components).T                    # reference AoS -> SoA
        return [np.ascontiguousarray(a[c]) for c in range(f.components)]
    stride = f.comp_stride or npts
    return [a[c * stride:c * stride + npts] for c in range(f.components)]


def encode_sem_frame(b: SemBlock, out: bytearray | None = None) -> memoryview:
    """One framed SemBlockPayload (header + payload), written into `out`
    (reused when large enough) and returned as a memoryview of it."""
    npts = b.point_count
    head = struct.pack("<qqqB", b.element_offset, b.n_elements, b.n_elements_global, b.order)
    parts: list = [head, b.x, b.y, b.z, struct.pack("<I", len(b.fields))]
    for f in b.fields:
        if f.association != POINT:
            raise ValueError(f"field {f.name!r}: SEM blocks carry point fields only")
        name = f.name.encode("utf-8")
        parts.append(struct.pack("<H", len(name)) + name + struct.pack("<BIQ", 0, f.components, f.components * npts))
        parts.extend(_soa(f, npts))

    def size(p) -> int:
        if isinstance(p, bytes):
            return len(p)
        if isinstance(p, tuple):                               # (device ptr, n)
            return 8 * p[1]
        if is_device_array(p):
            return 8 * npts
        return np.asarray(p).nbytes

    payload = sum(size(p) for p in parts)
    total = HEADER.size + payload
    if out is None or len(out) < total:
        out = bytearray(total)
    base = ctypes.addressof((ctypes.c_char * len(out)).from_buffer(out))
    off = 0

    def put(p):
        nonlocal off
        n = size(p)
        if isinstance(p, bytes):
            ctypes.memmove(base + off, p, n)
        elif isinstance(p, tuple):
            N.call("nkb_memcpy", base + off, p[0], n, 2, None)
        elif is_device_array(p):
            N.call("nkb_memcpy", base + off, device_ptr(p), n, 2, None)
        else:
            a = np.ascontiguousarray(p, dtype="<f8")
            ctypes.memmove(base + off, a.ctypes.data, n)
        off += n

    put(HEADER.pack(MAGIC, VERSION, TAG_SEM_BLOCK, payload))
    for p in parts:
        put(p)
    if any(isinstance(p, tuple) or is_device_array(p) for p in parts):
        N.call("nkb_stream_sync", None)
    return memoryview(out)[:total]


def decode_sem_frame(buf) -> SemBlock:
    """Inverse of encode_sem_frame (host arrays, SoA fields with comp_stride)."""
    buf = bytes(buf)
    if len(buf) < HEADER.size:
        raise ProtocolError("truncated frame header")
    magic, ver, tag, n = HEADER.unpack_from(buf, 0)
    if magic != MAGIC or ver != VERSION:
        raise ProtocolError(f"bad frame magic/version {magic!r}/{ver}")
    if tag != TAG_SEM_BLOCK:
        raise ProtocolError(f"not a SEM block frame (tag {tag:#x})")
    if len(buf) - HEADER.size != n:
        raise ProtocolError(f"payload length {len(buf) - HEADER.size} != declared {n}")
    try:
        pos = HEADER.size
        e_off, E, Eg, order = struct.unpack_from("<qqqB", buf, pos)
        pos += 25
        npts = E * (order + 1) ** 3

        def take(count):
            nonlocal pos
            end = pos + 8 * count
            if end > len(buf):
                raise ProtocolError("truncated SEM payload")
            a = np.frombuffer(buf, dtype="<f8", count=count, offset=pos).astype(np.float64)
            pos = end
            return a

        x, y, z = take(npts), take(npts), take(npts)
        (nf,) = struct.unpack_from("<I", buf, pos)
        pos += 4
        fields = []
        for _ in range(nf):
            (ln,) = struct.unpack_from("<H", buf, pos)
            pos += 2
            name = buf[pos:pos + ln].decode("utf-8")
            pos += ln
            assoc, comps, count = struct.unpack_from("<BIQ", buf, pos)
            pos += 13
            if assoc != 0 or count != comps * npts:
                raise ProtocolError(f"field {name!r}: bad association or value count")
            fields.append(FieldArray(name, POINT, comps, take(count), comp_stride=npts))
        if pos != len(buf):
            raise ProtocolError(f"{len(buf) - pos} trailing bytes in SEM payload")
    except struct.error as e:
        raise ProtocolError(f"truncated SEM payload: {e}") from e
    return SemBlock(E, x, y, z, order=order, fields=tuple(fields), element_offset=e_off, n_elements_global=Eg)
