"""Checkpoint files: legacy VTK, as the reference writes them.

Two layouts:

* SEM partitions (the in situ path): ``DATASET UNSTRUCTURED_GRID`` with the
  linear sub-hex mesh of R11 (GetMesh) and any AddArray arrays as point data.
  Every binary section (points, cells, cell types, arrays) is encoded
  big-endian ON THE GPU by ``nkb_encode_be`` and copied once into pinned host
  memory; Python only lays out the ASCII section headers.
* Structured blocks (the reference's own data model): ``DATASET
  STRUCTURED_POINTS`` in exactly the reference's layout (pkg/src/nekmini/
  sinks.py:1-21 module doc, _encode_vtk :76-102), so files are
  byte-identical and read back bit-exactly (checkpoint_read, :105-183).

File names follow checkpoint_filename (sinks.py:56-57).
"""
from __future__ import annotations

import ctypes
import re
from pathlib import Path

import numpy as np

from . import _native as N
from .data_model import CELL, POINT, Block, FieldArray, Snapshot
from .device import DeviceArray, PinnedBuffer

VTK_HEADER = "# vtk DataFile Version 3.0"
_SECTION = {POINT: "POINT_DATA", CELL: "CELL_DATA"}


class CheckpointFormatError(ValueError):
    """A checkpoint file is malformed or truncated (sinks.py:45-46)."""


def checkpoint_filename(step: int, blk: int) -> str:
    return f"step{step:06d}_blk{blk:03d}.vtk"


# ---------------------------------------------------------------- structured


def _g17(x: float) -> str:
    return f"{x:.17g}"


def encode_structured_vtk(block: Block, step: int, producer: int, time: float, fmt: str = "binary") -> bytes:
    """One structured block as a legacy-VTK STRUCTURED_POINTS file."""
    if fmt not in ("ascii", "binary"):
        raise ValueError(f"format must be 'ascii' or 'binary', got {fmt!r}")
    ni, nj, nk = block.dims
    head = [
        VTK_HEADER,
        f"nekmini step={step} producer={producer} time={_g17(time)} extents={' '.join(map(str, block.extents))}",
        fmt.upper(),
        "DATASET STRUCTURED_POINTS",
        f"DIMENSIONS {ni} {nj} {nk}",
        "ORIGIN " + " ".join(map(_g17, block.origin)),
        "SPACING " + " ".join(map(_g17, block.spacing)),
    ]
    parts = [("\n".join(head) + "\n").encode("ascii")]
    for assoc in (POINT, CELL):
        group = [f for f in block.fields if f.association == assoc]
        if not group:
            continue
        count = block.entity_count(assoc)
        parts.append(f"{_SECTION[assoc]} {count}\nFIELD FieldData {len(group)}\n".encode("ascii"))
        for f in group:
            parts.append(f"{f.name} {f.components} {count} double\n".encode("ascii"))
            vals = np.asarray(f.values, dtype=np.float64)
            if fmt == "binary":
                parts.append(vals.astype(">f8").tobytes())
            else:
                txt = [_g17(float(v)) for v in vals]
                parts.append(b"".join((" ".join(txt[i:i + 9]) + "\n").encode("ascii") for i in range(0, len(txt), 9)))
            parts.append(b"\n")
    return b"".join(parts)


def checkpoint_write(s: Snapshot, directory, fmt: str = "binary") -> tuple[list[Path], int]:
    """One file per block; (paths, total bytes) (sinks.py:60-73)."""
    if fmt not in ("ascii", "binary"):
        raise ValueError(f"format must be 'ascii' or 'binary', got {fmt!r}")
    paths, total = [], 0
    for bi, b in enumerate(s.blocks):
        if not b.fields:
            raise ValueError(f"block {bi} has no fields to checkpoint")
        blk = s.producer_id if len(s.blocks) == 1 else s.producer_id + bi
        p = Path(directory) / checkpoint_filename(s.step, blk)
        data = encode_structured_vtk(b, s.step, blk, s.time, fmt)
        p.write_bytes(data)
        paths.append(p)
        total += len(data)
    return paths, total


class _Cursor:
    def __init__(self, raw: bytes):
        self.raw, self.pos = raw, 0

    def line(self) -> str:
        nl = self.raw.find(b"\n", self.pos)
        if nl < 0:
            raise CheckpointFormatError("truncated header")
        out = self.raw[self.pos:nl].decode("ascii")
        self.pos = nl + 1
        return out

    def take(self, nbytes: int, what: str) -> bytes:
        end = self.pos + nbytes
        if end > len(self.raw):
            raise CheckpointFormatError(f"truncated payload for {what}")
        out = self.raw[self.pos:end]
        self.pos = end
        return out

    def skip_newlines(self):
        while self.pos < len(self.raw) and self.raw[self.pos:self.pos + 1] == b"\n":
            self.pos += 1

    def done(self) -> bool:
        return self.pos >= len(self.raw)


_TITLE = re.compile(r"nekmini step=(\d+) producer=(\d+) time=(\S+) extents=" + " ".join([r"(-?\d+)"] * 6))


def checkpoint_read(path) -> Snapshot:
    """Inverse of checkpoint_write for one structured file (sinks.py:105-183)."""
    cur = _Cursor(Path(path).read_bytes())
    if cur.line() != VTK_HEADER:
        raise CheckpointFormatError("not a legacy VTK file")
    m = _TITLE.match(cur.line())
    mode = cur.line()
    if mode not in ("BINARY", "ASCII"):
        raise CheckpointFormatError(f"unsupported data mode {mode!r}")
    ds = cur.line()
    if ds != "DATASET STRUCTURED_POINTS":
        raise CheckpointFormatError(f"unsupported dataset type {ds!r}")
    dims = tuple(int(v) for v in cur.line().split()[1:4])
    origin = tuple(float(v) for v in cur.line().split()[1:4])
    spacing = tuple(float(v) for v in cur.line().split()[1:4])
    if m:
        step, producer, t = int(m.group(1)), int(m.group(2)), float(m.group(3))
        extents = tuple(int(m.group(i)) for i in range(4, 10))
    else:
        step, producer, t = 0, 0, 0.0
        extents = (0, dims[0] - 1, 0, dims[1] - 1, 0, dims[2] - 1)
    fields = []
    while True:
        cur.skip_newlines()
        if cur.done():
            break
        sec = cur.line().split()
        assoc = POINT if sec[0] == "POINT_DATA" else CELL
        fl = cur.line().split()
        if fl[0] != "FIELD":
            raise CheckpointFormatError(f"expected FIELD, got {fl[0]!r}")
        for _ in range(int(fl[2])):
            name, comps, count, dtype = cur.line().split()
            if dtype != "double":
                raise CheckpointFormatError(f"unsupported dtype {dtype!r}")
            n = int(comps) * int(count)
            if mode == "BINARY":
                vals = np.frombuffer(cur.take(8 * n, f"field {name!r}"), dtype=">f8").astype(np.float64)
            else:
                got: list[float] = []
                while len(got) < n:
                    if cur.done():
                        raise CheckpointFormatError(f"truncated payload for field {name!r}")
                    got.extend(float(v) for v in cur.line().split())
                vals = np.array(got[:n])
            fields.append(FieldArray(name, assoc, int(comps), vals))
            if cur.raw[cur.pos:cur.pos + 1] == b"\n":
                cur.pos += 1
    return Snapshot(time=t, step=step, producer_id=producer, blocks=(Block(origin, spacing, extents, tuple(fields)),))


# ---------------------------------------------------------------------- SEM


class SemVtkWriter:
    """SEM partition -> legacy-VTK UNSTRUCTURED_GRID bytes, GPU-encoded.

    Reusable across steps: keeps one device scratch (largest section) and one
    pinned host buffer (whole file)."""

    def __init__(self, ctx):
        self.ctx = ctx
        self._scratch: DeviceArray | None = None
        self._host: PinnedBuffer | None = None

    def _size(self, what: str) -> int:
        n = ctypes.c_int64()
        N.call("nkb_encode_be", self.ctx.handle, what.encode(), None, 0, ctypes.byref(n), None)
        return int(n.value)

    def encode(self, adaptor, arrays, step: int, producer: int, time: float) -> memoryview:
        md = adaptor.get_mesh_metadata()
        npts, ncells = md.n_points, md.n_cells
        comps = {a: self.ctx.array_components(a) for a in arrays}
        title = (f"nekb200 step={step} producer={producer} time={_g17(time)} "
                 f"elements={md.n_elements} order={md.order}")
        plan: list[bytes | str] = [
            f"{VTK_HEADER}\n{title}\nBINARY\nDATASET UNSTRUCTURED_GRID\nPOINTS {npts} double\n".encode(),
            "POINTS", f"\nCELLS {ncells} {9 * ncells}\n".encode(), "CELLS",
            f"\nCELL_TYPES {ncells}\n".encode(), "CELL_TYPES", b"\n",
        ]
        if arrays:
            plan.append(f"POINT_DATA {npts}\nFIELD FieldData {len(arrays)}\n".encode())
            for a in arrays:
                plan += [f"{a} {comps[a]} {npts} double\n".encode(), a, b"\n"]
        sizes = [len(p) if isinstance(p, bytes) else self._size(p) for p in plan]
        total, biggest = sum(sizes), max([s for p, s in zip(plan, sizes) if isinstance(p, str)] + [8])
        if self._scratch is None or self._scratch.nbytes < biggest:
            self._scratch = DeviceArray.empty(self.ctx, ((biggest + 7) // 8,), np.float64)
        if self._host is None or self._host.nbytes < total:
            self._host = PinnedBuffer(total)
        off = 0
        for p, sz in zip(plan, sizes):
            if isinstance(p, bytes):
                ctypes.memmove(self._host.ptr + off, p, sz)
            elif sz:
                n = ctypes.c_int64()
                N.call("nkb_encode_be", self.ctx.handle, p.encode(), self._scratch.ptr, self._scratch.nbytes,
                       ctypes.byref(n), None)
                N.call("nkb_memcpy", self._host.ptr + off, self._scratch.ptr, sz, 2, None)
            off += sz
        N.call("nkb_stream_sync", None)
        return memoryview((ctypes.c_ubyte * total).from_address(self._host.ptr)).cast("B")


def read_sem_vtk(path) -> dict:
    """Parse a file written by SemVtkWriter: title fields, points (n, 3),
    cells (m, 8) int64, types (m,), arrays {name: (n, comps) or (n,)}."""
    cur = _Cursor(Path(path).read_bytes())
    if cur.line() != VTK_HEADER:
        raise CheckpointFormatError("not a legacy VTK file")
    title = dict(kv.split("=", 1) for kv in cur.line().split()[1:])
    if cur.line() != "BINARY" or cur.line() != "DATASET UNSTRUCTURED_GRID":
        raise CheckpointFormatError("not a binary UNSTRUCTURED_GRID file")
    out: dict = {"step": int(title["step"]), "producer": int(title["producer"]), "time": float(title["time"]),
                 "n_elements": int(title["elements"]), "order": int(title["order"]), "arrays": {}}
    _, npts, _ = cur.line().split()
    npts = int(npts)
    out["points"] = np.frombuffer(cur.take(24 * npts, "POINTS"), ">f8").astype(np.float64).reshape(npts, 3)
    cur.skip_newlines()
    _, ncells, size = cur.line().split()
    ncells = int(ncells)
    cells = np.frombuffer(cur.take(4 * int(size), "CELLS"), ">i4").astype(np.int64).reshape(ncells, 9)
    if ncells and not (cells[:, 0] == 8).all():
        raise CheckpointFormatError("non-hexahedral cell")
    out["cells"] = cells[:, 1:]
    cur.skip_newlines()
    _, nt = cur.line().split()
    out["types"] = np.frombuffer(cur.take(4 * int(nt), "CELL_TYPES"), ">i4").astype(np.int64)
    cur.skip_newlines()
    if not cur.done():
        cur.line()                                   # POINT_DATA n
        k = int(cur.line().split()[2])               # FIELD FieldData k
        for _ in range(k):
            name, comps, count, _ = cur.line().split()
            n, c = int(count), int(comps)
            v = np.frombuffer(cur.take(8 * n * c, name), ">f8").astype(np.float64)
            out["arrays"][name] = v.reshape(n, c) if c > 1 else v
            cur.skip_newlines()
    return out
