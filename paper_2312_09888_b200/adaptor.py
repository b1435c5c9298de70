"""SENSEI-style DataAdaptor for NekRS-layout spectral-element data.

Mirrors the paper's `nek_sensei::DataAdaptor` surface (PAPER.md:141-150:
Initialize / GetNumberOfMeshes / GetMeshMetadata / GetMesh / AddArray) on top
of libnekb200.  It replaces the reference's adaptor step
`solver.snapshot_of` (reference solver.py:282-305), which copies the
solver-native layout into VTK-ordered point arrays on the host: here the VTK
view (linear sub-hexes, AoS arrays) is produced on the GPU, on request, from
the device-resident SEM fields -- and the in situ analysis never needs it
materialised at all (the fused kernel reads the SEM layout directly).

Host (numpy) inputs are accepted and uploaded into adaptor-owned device
buffers that are reused across steps (the end-to-end path a host-resident
solver would take).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .context import Context
from .data_model import POINT, FieldArray, MeshMetadata, SemBlock, Snapshot, validate_snapshot
from .device import DeviceArray, device_ptr, is_device_array


@dataclass
class UnstructuredGrid:
    """GetMesh result: VTK unstructured grid of linear sub-hexes, on device."""

    points: DeviceArray | None        # (n_points, 3) float64 AoS
    connectivity: DeviceArray | None  # (n_cells, 8) int64, VTK_HEXAHEDRON order
    offsets: DeviceArray | None       # (n_cells + 1,) int64
    types: DeviceArray | None         # (n_cells,) uint8 == 12
    n_points: int
    n_cells: int


def _read_only(a) -> bool:
    return isinstance(a, np.ndarray) and not a.flags.writeable


class SemDataAdaptor:
    """DataAdaptor over one SemBlock per rank (NekRS partition)."""

    MESH_NAME = "mesh"

    def __init__(self, ctx: Context | None = None, device: int = 0, velocity: str = "velocity"):
        self.ctx = ctx if ctx is not None else Context(device)
        self.velocity = velocity
        self.ctx.set_velocity_name(velocity)
        self._block: SemBlock | None = None
        self._staging: dict[str, DeviceArray] = {}
        self._fields: dict[str, FieldArray] = {}
        self._coords = None
        self._gid = None
        self._segments: dict[str, tuple[int, int, int]] = {}   # name -> (ptr, ncomp, comp_stride)
        self.time = 0.0
        self.step = 0
        self.h2d_bytes = 0

    # ---- Initialize(nek_data) ------------------------------------------------------
    def initialize(self, snapshot: Snapshot) -> None:
        """Bind a snapshot whose single block is a SemBlock (host or device arrays)."""
        v = validate_snapshot(snapshot)
        if v:
            raise ValueError(f"invalid snapshot: {v}")
        if len(snapshot.blocks) != 1 or not isinstance(snapshot.blocks[0], SemBlock):
            raise ValueError("the SEM adaptor takes exactly one SemBlock per rank (single mesh, SPEC.md:79)")
        b: SemBlock = snapshot.blocks[0]
        self.time, self.step = float(snapshot.time), int(snapshot.step)
        self.h2d_bytes = 0
        npts = b.point_count
        # Static mesh (NekRS without a moving mesh): when the block carries the
        # very same read-only host coordinate arrays as last step, they are
        # already resident and the library keeps its geometry cache.  Any
        # other host coordinates are re-uploaded and the cache is dropped.
        coords = (b.x, b.y, b.z)
        static = (self._coords is not None and all(a is p for a, p in zip(coords, self._coords))
                  and all(_read_only(a) for a in coords) and "__x" in self._staging)
        if static:
            x, y, z = (self._staging[k] for k in ("__x", "__y", "__z"))
        else:
            x = self._dev("__x", b.x, npts)
            y = self._dev("__y", b.y, npts)
            z = self._dev("__z", b.z, npts)
        self.ctx.mesh_set(b.n_elements, x, y, z, order=b.order, element_offset=b.element_offset,
                          n_elements_global=b.n_elements_global)
        if not static and not all(is_device_array(a) for a in coords):
            self.ctx.mesh_modified()
        self._coords = coords
        gid = b.global_ids
        if gid is None:
            self._gid = None
        elif not (static and gid is self._gid):
            # global node ids: the DSSUM gather-scatter (nkb_mesh_set_global_ids)
            if is_device_array(gid):
                dg = gid
            else:
                a = np.ascontiguousarray(gid, dtype=np.int64).ravel()
                if a.size != npts:
                    raise ValueError(f"global_ids: expected {npts} ids, got {a.size}")
                dg = self._staging.get("__gid")
                if dg is None or dg.size != a.size:
                    dg = DeviceArray.empty(self.ctx, (a.size,), np.int64)
                    self._staging["__gid"] = dg
                dg.upload(a, sync=False)
                self.h2d_bytes += a.nbytes
            self.ctx.mesh_set_global_ids(dg)
            self._gid = gid
        self.ctx.field_clear()
        self._fields = {}
        self._segments = {}
        for f in b.fields:
            if f.association != POINT:
                raise ValueError(f"field {f.name!r}: only point fields exist on the SEM mesh")
            self._bind_field(f, npts)
            self._fields[f.name] = f
        self._block = b

    def _dev(self, key: str, arr, n: int, ncomp: int = 1):
        if is_device_array(arr):
            return arr
        a = np.ascontiguousarray(arr, dtype=np.float64).ravel()
        if a.size != n * ncomp:
            raise ValueError(f"{key}: expected {n * ncomp} values, got {a.size}")
        d = self._staging.get(key)
        if d is None or d.size != a.size:
            d = DeviceArray.empty(self.ctx, (a.size,), np.float64)
            self._staging[key] = d
        d.upload(a, sync=False)
        self.h2d_bytes += a.nbytes
        return d

    def _set(self, name: str, base, ncomp: int, stride: int) -> None:
        self.ctx.field_set(name, base, ncomp, stride)
        self._segments[name] = (device_ptr(base), ncomp, stride)

    def field_segment(self, name: str) -> tuple[int, int, int, int]:
        """(device ptr, n_points, ncomp, comp_stride) of a bound point field."""
        if name not in self._segments:
            raise ValueError(f"no field named {name!r}")
        ptr, nc, st = self._segments[name]
        return ptr, self._require().point_count, nc, st

    def _bind_field(self, f: FieldArray, npts: int) -> None:
        if isinstance(f.values, tuple):  # one device (or host) array per component
            comps = [self._dev(f"{f.name}#{c}", f.values[c], npts) for c in range(f.components)]
            if f.components == 1:
                self._set(f.name, comps[0], 1, npts)
                return
            # components must be evenly spaced for the ABI's (base, stride) form
            ptrs = [device_ptr(c) for c in comps]
            stride = (ptrs[1] - ptrs[0]) // 8 if len(ptrs) > 1 else npts
            if all(ptrs[c] == ptrs[0] + 8 * stride * c for c in range(len(ptrs))) and stride >= npts:
                self._set(f.name, ptrs[0], f.components, stride)
                return
            # not evenly spaced: gather into one staging array (D2D)
            d = self._staging.get(f.name)
            if d is None or d.size != f.components * npts:
                d = DeviceArray.empty(self.ctx, (f.components * npts,), np.float64)
                self._staging[f.name] = d
            for c, p in enumerate(ptrs):
                N.call("nkb_memcpy", d.ptr + 8 * c * npts, p, 8 * npts, 3, None)
            self._set(f.name, d, f.components, npts)
            return
        if is_device_array(f.values):
            stride = f.comp_stride or npts
            self._set(f.name, f.values, f.components, stride)
            return
        # host values: component-fastest AoS (reference layout) or SoA with comp_stride
        a = np.asarray(f.values, dtype=np.float64)
        if f.components > 1 and not f.comp_stride:
            a = np.ascontiguousarray(a.reshape(npts, f.components).T)   # AoS -> SoA
            d = self._dev(f.name, a, npts, f.components)
            self._set(f.name, d, f.components, npts)
        else:
            stride = f.comp_stride or npts
            n = (f.components - 1) * stride + npts
            d = self._dev(f.name, a[:n], n)
            self._set(f.name, d, f.components, stride)

    # ---- GetNumberOfMeshes / GetMeshMetadata ------------------------------------------
    def get_number_of_meshes(self) -> int:
        return 1

    def get_mesh_metadata(self, index: int = 0) -> MeshMetadata:
        if index != 0:
            raise IndexError("single mesh (SPEC.md:79)")
        b = self._require()
        m = self.ctx.metadata()
        descriptors = tuple((f.name, f.association, f.components) for f in b.fields)
        return MeshMetadata(
            self.MESH_NAME, (0, 0, 0, 0, 0, 0), descriptors, 1,
            n_elements=int(m.n_elements), order=int(m.order), n_points=int(m.n_points),
            n_cells=int(m.n_cells), cell_type=int(m.cell_type), element_offset=int(m.element_offset),
            n_elements_global=int(m.n_elements_global),
        )

    # ---- GetMesh ---------------------------------------------------------------------
    def get_mesh(self, mesh_name: str = MESH_NAME, structure_only: bool = False) -> UnstructuredGrid:
        if mesh_name != self.MESH_NAME:
            raise KeyError(f"no mesh named {mesh_name!r}")
        self._require()
        m = self.ctx.metadata()
        npts, ncells = int(m.n_points), int(m.n_cells)
        pts = None if structure_only else DeviceArray.empty(self.ctx, (npts, 3), np.float64)
        conn = DeviceArray.empty(self.ctx, (ncells, 8), np.int64)
        offs = DeviceArray.empty(self.ctx, (ncells + 1,), np.int64)
        types = DeviceArray.empty(self.ctx, (ncells,), np.uint8)
        self.ctx.get_mesh(pts, conn, offs, types)
        N.call("nkb_stream_sync", None)
        return UnstructuredGrid(pts, conn, offs, types, npts, ncells)

    # ---- AddArray --------------------------------------------------------------------
    def add_array(self, mesh_name: str, association: str, array_name: str) -> FieldArray:
        """VTK AoS point array `array_name` (registered field, '<vec>:mag', 'Q',
        'vorticity', 'vorticity:mag') as a device-resident FieldArray."""
        if mesh_name != self.MESH_NAME:
            raise KeyError(f"no mesh named {mesh_name!r}")
        if association != POINT:
            raise ValueError("only point arrays exist on the SEM mesh")
        self._require()
        npts = int(self.ctx.metadata().n_points)
        nc = self.ctx.array_components(array_name)
        out = DeviceArray.empty(self.ctx, (npts * nc,), np.float64)
        self.ctx.add_array(array_name, out)
        N.call("nkb_stream_sync", None)
        return FieldArray(array_name, POINT, nc, out)

    def mesh_modified(self) -> None:
        """The bound coordinates were edited in place (moving mesh): the
        geometry cache is rebuilt on the next gradient step."""
        self.ctx.mesh_modified()

    def release_data(self) -> None:
        self._block = None
        self._fields = {}

    def _require(self) -> SemBlock:
        if self._block is None:
            raise RuntimeError("DataAdaptor used before initialize()")
        return self._block
