"""Data model: the reference's structured-grid contract plus the SEM mesh.

Mirrors `nekmini.data_model` (reference pkg/src/nekmini/data_model.py) so the
reference's snapshots and ours are interchangeable at the sink boundary:

* `FieldArray` (:27-55), `Block` (:58-95), `Snapshot` (:98-108),
  `MeshMetadata`/`metadata_of` (:111-128), `validate_snapshot` (:131-175),
  `SchemaMismatch` (:178-179), `assemble_global` (:188-225) -- same fields,
  same invariants, same messages.
* Divergence (deliberate, north star): a FieldArray's ``values`` may be a
  DEVICE array (torch CUDA tensor, DeviceArray, anything with
  ``__cuda_array_interface__``), which is borrowed, not copied.  Host values
  keep the reference's copy + read-only semantics.
* New: `SemBlock` -- an order-N spectral-element block (E elements, (N+1)^3
  GLL nodes each, element-local layout i fastest; NekRS convention) carrying
  SoA point fields.  It is what the in situ path consumes.

Array layout convention (reference data_model.py:8-14): flat float64,
component fastest, then x, y, z: ``flat = c + components*(i + ni*(j + nj*k))``.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .device import is_device_array

POINT = "point"
CELL = "cell"


def _values_size(v) -> int:
    if is_device_array(v):
        shape = getattr(v, "shape", None)
        if shape is None:
            shape = v.__cuda_array_interface__["shape"]
        return int(np.prod(tuple(shape))) if len(tuple(shape)) else 1
    return int(np.asarray(v).size)


@dataclass(frozen=True)
class FieldArray:
    """A named array attached to a block (reference data_model.py:27-55).

    Host values: flat, C-contiguous float64 copy, read-only.  Device values
    (SEM path): borrowed; for a SemBlock, a multi-component field is either a
    tuple of per-component device arrays or one device array of
    ``components * comp_stride`` doubles (NekRS fieldOffset layout).
    """

    name: str
    association: str  # POINT or CELL
    components: int
    values: object
    comp_stride: int = 0

    def __post_init__(self):
        v = self.values
        if isinstance(v, tuple):
            if len(v) != self.components:
                raise ValueError("one device array per component expected")
            return
        if is_device_array(v):
            return
        if (isinstance(v, np.ndarray) and v.dtype == np.float64 and v.flags.c_contiguous
                and not v.flags.writeable):
            # already immutable: alias it (lets pinned host staging reach the
            # GPU without a pageable copy); anything else is copied + frozen
            object.__setattr__(self, "values", v.reshape(-1))
            return
        vals = np.array(v, dtype=np.float64, copy=True).ravel()
        vals.setflags(write=False)
        object.__setattr__(self, "values", vals)

    @property
    def on_device(self) -> bool:
        v = self.values
        return isinstance(v, tuple) or is_device_array(v)

    @property
    def size(self) -> int:
        v = self.values
        if isinstance(v, tuple):
            return sum(_values_size(c) for c in v)
        return _values_size(v)

    def __eq__(self, other):
        if not isinstance(other, FieldArray):
            return NotImplemented
        if self.on_device or other.on_device:
            return self is other
        return (
            self.name == other.name
            and self.association == other.association
            and self.components == other.components
            and self.values.shape == other.values.shape
            and bool(np.all(self.values == other.values))
        )

    __hash__ = None


@dataclass(frozen=True)
class Block:
    """One structured-points block (reference data_model.py:58-95)."""

    origin: tuple[float, float, float]
    spacing: tuple[float, float, float]
    extents: tuple[int, int, int, int, int, int]
    fields: tuple[FieldArray, ...] = field(default_factory=tuple)

    def __post_init__(self):
        object.__setattr__(self, "origin", tuple(float(x) for x in self.origin))
        object.__setattr__(self, "spacing", tuple(float(x) for x in self.spacing))
        object.__setattr__(self, "extents", tuple(int(x) for x in self.extents))
        object.__setattr__(self, "fields", tuple(self.fields))

    @property
    def dims(self) -> tuple[int, int, int]:
        e = self.extents
        return (e[1] - e[0] + 1, e[3] - e[2] + 1, e[5] - e[4] + 1)

    @property
    def point_count(self) -> int:
        ni, nj, nk = self.dims
        return ni * nj * nk

    @property
    def cell_count(self) -> int:
        return int(np.prod([max(n - 1, 1) if n > 0 else 0 for n in self.dims]))

    def entity_count(self, association: str) -> int:
        return self.point_count if association == POINT else self.cell_count

    def field_named(self, name: str) -> FieldArray:
        for f in self.fields:
            if f.name == name:
                return f
        raise KeyError(f"no field named {name!r}")


@dataclass(frozen=True)
class SemBlock:
    """Order-N hexahedral spectral elements on the device (NekRS layout).

    x, y, z: device arrays of E*(N+1)^3 doubles (element-major, node i
    fastest).  `element_offset` / `n_elements_global` describe this rank's
    contiguous slice of the global mesh (NekRS-style partition).
    """

    n_elements: int
    x: object
    y: object
    z: object
    order: int = 7
    fields: tuple[FieldArray, ...] = field(default_factory=tuple)
    element_offset: int = 0
    n_elements_global: int = 0
    global_ids: object = None     # optional int64 global node ids (NekRS mesh->globalIds): enables DSSUM

    def __post_init__(self):
        object.__setattr__(self, "fields", tuple(self.fields))
        if self.n_elements_global == 0:
            object.__setattr__(self, "n_elements_global", int(self.n_elements))

    @property
    def nodes_per_element(self) -> int:
        return (self.order + 1) ** 3

    @property
    def cells_per_element(self) -> int:
        return self.order ** 3

    @property
    def point_count(self) -> int:
        return self.n_elements * self.nodes_per_element

    @property
    def cell_count(self) -> int:
        return self.n_elements * self.cells_per_element

    def entity_count(self, association: str) -> int:
        return self.point_count if association == POINT else self.cell_count

    def field_named(self, name: str) -> FieldArray:
        for f in self.fields:
            if f.name == name:
                return f
        raise KeyError(f"no field named {name!r}")


@dataclass(frozen=True)
class Snapshot:
    """The unit handed to analyses (reference data_model.py:98-108)."""

    time: float
    step: int
    producer_id: int
    blocks: tuple

    def __post_init__(self):
        object.__setattr__(self, "blocks", tuple(self.blocks))


@dataclass(frozen=True)
class MeshMetadata:
    """GetMeshMetadata (reference data_model.py:111-116) + SEM descriptors."""

    mesh_name: str
    global_extents: tuple[int, int, int, int, int, int]
    field_descriptors: tuple[tuple[str, str, int], ...]
    block_count: int
    # SEM additions (zero for structured snapshots)
    n_elements: int = 0
    order: int = 0
    n_points: int = 0
    n_cells: int = 0
    cell_type: int = 0          # 12 = VTK_HEXAHEDRON
    element_offset: int = 0
    n_elements_global: int = 0


def metadata_of(s: Snapshot, mesh_name: str = "mesh") -> MeshMetadata:
    """Describe a snapshot (reference data_model.py:119-128)."""
    b0 = s.blocks[0]
    descriptors = tuple((f.name, f.association, f.components) for f in b0.fields)
    if isinstance(b0, SemBlock):
        E = sum(b.n_elements for b in s.blocks)
        return MeshMetadata(
            mesh_name, (0, 0, 0, 0, 0, 0), descriptors, len(s.blocks),
            n_elements=E, order=b0.order, n_points=sum(b.point_count for b in s.blocks),
            n_cells=sum(b.cell_count for b in s.blocks), cell_type=12,
            element_offset=b0.element_offset, n_elements_global=b0.n_elements_global,
        )
    ext = np.array([b.extents for b in s.blocks])
    global_extents = (
        int(ext[:, 0].min()), int(ext[:, 1].max()),
        int(ext[:, 2].min()), int(ext[:, 3].max()),
        int(ext[:, 4].min()), int(ext[:, 5].max()),
    )
    return MeshMetadata(mesh_name, global_extents, descriptors, len(s.blocks))


def validate_snapshot(s: Snapshot) -> list[str]:
    """Every type invariant; [] when valid; never raises (data_model.py:131-175).

    SEM blocks: positive order, coordinate/field lengths = E*(N+1)^3 (per
    component), unique names, same schema across blocks.
    """
    violations: list[str] = []
    if len(s.blocks) == 0:
        return ["snapshot has no blocks"]
    if s.step < 0:
        violations.append("negative step")
    schema = None
    for bi, b in enumerate(s.blocks):
        if isinstance(b, SemBlock):
            if b.order < 1:
                violations.append(f"block {bi}: order < 1")
                continue
            if b.n_elements < 0:
                violations.append(f"block {bi}: negative element count")
                continue
            for nm, arr in (("x", b.x), ("y", b.y), ("z", b.z)):
                if b.n_elements and _values_size(arr) < b.point_count:
                    violations.append(f"block {bi}: coordinate {nm} shorter than {b.point_count}")
        else:
            e = b.extents
            if e[1] < e[0] or e[3] < e[2] or e[5] < e[4]:
                violations.append(f"block {bi}: inverted extents {e}")
                continue
            for ax, sp in enumerate(b.spacing):
                if not sp > 0:
                    violations.append(f"block {bi}: non-positive spacing on axis {ax}")
        seen: set[str] = set()
        for f in b.fields:
            if not f.name:
                violations.append(f"block {bi}: empty field name")
            if f.name in seen:
                violations.append(f"block {bi}: duplicate field name {f.name!r}")
            seen.add(f.name)
            if f.association not in (POINT, CELL):
                violations.append(f"block {bi}, field {f.name!r}: bad association")
                continue
            if f.components < 1:
                violations.append(f"block {bi}, field {f.name!r}: components < 1")
                continue
            n_ent = b.entity_count(f.association)
            expected = f.components * n_ent
            if isinstance(b, SemBlock) and f.on_device and not isinstance(f.values, tuple) and f.components > 1:
                # one device array holding `components` runs, comp_stride apart (NekRS fieldOffset)
                need = (f.components - 1) * max(f.comp_stride, n_ent) + n_ent
                if f.size < need:
                    violations.append(
                        f"block {bi}, field {f.name!r}: field length mismatch "
                        f"(got {f.size}, expected >= {need})"
                    )
            elif isinstance(f.values, tuple):
                if any(_values_size(c) != n_ent for c in f.values):
                    violations.append(
                        f"block {bi}, field {f.name!r}: field length mismatch "
                        f"(got {[_values_size(c) for c in f.values]}, expected {n_ent} per component)"
                    )
            elif f.size != expected:
                violations.append(
                    f"block {bi}, field {f.name!r}: field length mismatch "
                    f"(got {f.size}, expected {expected})"
                )
        sig = tuple((f.name, f.association, f.components) for f in b.fields)
        if schema is None:
            schema = sig
        elif set(sig) != set(schema):
            violations.append(f"block {bi}: field schema differs from block 0")
    return violations


class SchemaMismatch(ValueError):
    pass


def _grid(f: FieldArray, dims: tuple[int, int, int]) -> np.ndarray:
    ni, nj, nk = dims
    return f.values.reshape(nk, nj, ni, f.components)


def assemble_global(blocks: list[Block], layout: str = "tile_x") -> Block:
    """Tile host blocks along x in producer order (data_model.py:188-225).

    The GPU renderer never materialises this: it samples the blocks in place
    through a column-prefix table (RenderSink / nkb_render_structured).  This
    host version keeps the reference's contract for callers that need it.
    """
    if layout != "tile_x":
        raise ValueError(f"unknown layout {layout!r}")
    if not blocks:
        raise ValueError("no blocks to assemble")
    if len(blocks) == 1:
        return blocks[0]
    first = blocks[0]
    check_assembly(blocks)
    ni_total = sum(b.dims[0] for b in blocks)
    e = first.extents
    global_extents = (e[0], e[0] + ni_total - 1, e[2], e[3], e[4], e[5])
    schema = tuple((f.name, f.association, f.components) for f in first.fields)
    out_fields = []
    for fi, (name, assoc, comps) in enumerate(schema):
        parts = [_grid(b.fields[fi], b.dims) for b in blocks]
        merged = np.concatenate(parts, axis=2)
        out_fields.append(FieldArray(name, assoc, comps, merged.ravel()))
    return Block(first.origin, first.spacing, global_extents, tuple(out_fields))


def check_assembly(blocks) -> None:
    """The validation half of assemble_global (data_model.py:202-210, :219-220)."""
    first = blocks[0]
    schema = tuple((f.name, f.association, f.components) for f in first.fields)
    for b in blocks[1:]:
        if tuple(b.spacing) != tuple(first.spacing):
            raise SchemaMismatch("spacing differs across blocks")
        if tuple((f.name, f.association, f.components) for f in b.fields) != schema:
            raise SchemaMismatch("field schema differs across blocks")
        if tuple(b.extents[2:]) != tuple(first.extents[2:]):
            raise SchemaMismatch("y/z extents differ across blocks")
    if len(blocks) > 1:
        for (name, assoc, comps) in schema:
            if assoc == CELL:
                raise SchemaMismatch("cell-centered tiling across blocks is unsupported")
