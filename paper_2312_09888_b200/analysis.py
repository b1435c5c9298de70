"""The in situ AnalysisAdaptor: SEM adaptor -> Q-criterion -> isosurface /
slice -> render -> sort-last composite, on the GPU.

This is the B200 stand-in for the Catalyst AnalysisAdaptor the paper drives
through SENSEI (`type="catalyst"`), whose desk-scale
analogue in the reference is `RenderSink.consume` -> `render`
(reference sinks.py:245-295, :327-351).  The colormap, its global-range rule,
the degenerate-range rule and the row-0-is-top orientation are the
reference's (sinks.py:201-213, :256-269).

Pipeline parameters come from the same kind of `<analysis .../>` attribute
map the reference's sinks take (params: dict[str, str], bridge.py:83-96):

    iso="Q=0.1;temperature=0.5"   up to 4 surfaces in total
    slice="y=0" | "0,1,0,0"       plane n.x = c ("axis=c" or "nx,ny,nz,c")
    field="temperature"           colour field ("velocity:mag", "Q", ...)
    width / height / vmin / vmax  as the reference's render sink
    view="+z" | "az,el"           orthographic camera direction (degrees)
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .context import Report

DEFAULT_ANCHORS = ((0.0, (59, 76, 192)), (0.5, (255, 255, 255)), (1.0, (180, 4, 38)))


@dataclass(frozen=True)
class Surface:
    kind: str                 # "iso" | "slice"
    field: str = ""           # iso field
    value: float = 0.0        # iso value / plane offset c
    normal: tuple[float, float, float] = (0.0, 0.0, 1.0)


@dataclass(frozen=True)
class Pipeline:
    surfaces: tuple[Surface, ...] = ()
    color_field: str = "velocity:mag"
    width: int = 256
    height: int = 256
    view: tuple[float, ...] | None = None     # 3x4 row-major (+ perspective row: 16); None -> auto
    view_dir: tuple[float, float] = (0.0, 90.0)   # azimuth, elevation (deg) for auto
    projection: str = "ortho"                 # auto camera: "ortho" or "perspective"
    fov: float = 30.0                         # perspective: vertical field of view (deg)
    vmin: float | None = None
    vmax: float | None = None
    anchors: tuple = DEFAULT_ANCHORS
    background: tuple[int, int, int, int] = (0, 0, 0, 0)
    emit_meta: bool = False
    composite: bool = True
    continuous: bool = False      # DSSUM-average Q / vorticity:mag first (needs SemBlock.global_ids)
    timing: bool = False

    def native(self, view: tuple[float, ...]) -> N.NkbPipeline:
        p = N.NkbPipeline()
        if len(self.surfaces) > N.NKB_MAX_SURFACES:
            raise ValueError(f"at most {N.NKB_MAX_SURFACES} surfaces")
        p.n_surfaces = len(self.surfaces)
        for k, s in enumerate(self.surfaces):
            ns = p.surfaces[k]
            if s.kind == "iso":
                ns.kind = N.NKB_SURF_ISO
                ns.field = s.field.encode()
            elif s.kind == "slice":
                ns.kind = N.NKB_SURF_SLICE
            else:
                raise ValueError(f"unknown surface kind {s.kind!r}")
            ns.value = float(s.value)
            for a in range(3):
                ns.normal[a] = float(s.normal[a])
        p.color_field = self.color_field.encode()
        p.width, p.height = int(self.width), int(self.height)
        if len(view) not in (12, 16):
            raise ValueError("view must have 12 values (3x4) or 16 (3x4 + perspective row)")
        for i in range(12):
            p.view[i] = float(view[i])
        for i in range(4):
            p.persp[i] = float(view[12 + i]) if len(view) == 16 else 0.0
        p.vmin = math.nan if self.vmin is None else float(self.vmin)
        p.vmax = math.nan if self.vmax is None else float(self.vmax)
        if tuple(self.anchors) == DEFAULT_ANCHORS:
            p.n_anchors = 0
        else:
            p.n_anchors = len(self.anchors)
            for i, (t, rgb) in enumerate(self.anchors):
                p.anchor_t[i] = float(t)
                for c in range(3):
                    p.anchor_rgb[i][c] = int(rgb[c])
        for c in range(4):
            p.background[c] = int(self.background[c])
        p.emit_meta = int(self.emit_meta)
        p.composite = int(self.composite)
        p.continuous = int(self.continuous)
        p.timing = int(self.timing)
        return p


def ortho_view(bounds, width: int, height: int, azimuth: float = 0.0, elevation: float = 90.0,
               margin: float = 1.05) -> tuple[float, ...]:
    """3x4 matrix mapping world (x,y,z,1) -> (column, row, depth in [0,1]).

    Fits the bounding sphere of `bounds` (xmin,xmax,ymin,ymax,zmin,zmax) in
    the image; row 0 is the top of the image (reference sinks.py:256-257),
    depth grows away from the camera.  elevation=90 looks down -z with +x
    right and +y up.
    """
    b = np.asarray(bounds, dtype=np.float64)
    c = np.array([(b[0] + b[1]) / 2, (b[2] + b[3]) / 2, (b[4] + b[5]) / 2])
    r = 0.5 * math.sqrt((b[1] - b[0]) ** 2 + (b[3] - b[2]) ** 2 + (b[5] - b[4]) ** 2)
    r = max(r, 1e-300) * margin
    az, el = math.radians(azimuth), math.radians(elevation)
    eye = np.array([math.cos(el) * math.cos(az), math.cos(el) * math.sin(az), math.sin(el)])
    fwd = -eye
    up0 = np.array([0.0, 1.0, 0.0]) if abs(eye[2]) > 0.999 else np.array([0.0, 0.0, 1.0])
    right = np.cross(fwd, up0)
    right /= np.linalg.norm(right)
    up = np.cross(right, fwd)
    s = min(width, height) / (2.0 * r)
    row0 = np.concatenate([s * right, [width / 2.0 - s * right.dot(c)]])
    row1 = np.concatenate([-s * up, [height / 2.0 + s * up.dot(c)]])
    row2 = np.concatenate([fwd / (2.0 * r), [0.5 - fwd.dot(c) / (2.0 * r)]])
    return tuple(float(v) for v in np.concatenate([row0, row1, row2]))


def perspective_view(bounds, width: int, height: int, azimuth: float = 0.0, elevation: float = 90.0,
                     fov: float = 30.0, margin: float = 1.05) -> tuple[float, ...]:
    """16 values: the 3x4 rows and the w row of a pinhole camera that sees
    the bounding sphere of `bounds` in a `fov`-degree cone from direction
    (azimuth, elevation).  (col, row, depth) = rows . X / (w . X): depth is
    0 on the near and 1 on the far side of the sphere, row 0 is the top."""
    b = np.asarray(bounds, dtype=np.float64)
    c = np.array([(b[0] + b[1]) / 2, (b[2] + b[3]) / 2, (b[4] + b[5]) / 2])
    r = 0.5 * math.sqrt((b[1] - b[0]) ** 2 + (b[3] - b[2]) ** 2 + (b[5] - b[4]) ** 2)
    r = max(r, 1e-300) * margin
    half = math.radians(fov) / 2.0
    az, el = math.radians(azimuth), math.radians(elevation)
    d = np.array([math.cos(el) * math.cos(az), math.cos(el) * math.sin(az), math.sin(el)])
    dist = r / math.sin(half)
    eye = c + dist * d
    fwd = -d
    up0 = np.array([0.0, 1.0, 0.0]) if abs(d[2]) > 0.999 else np.array([0.0, 0.0, 1.0])
    right = np.cross(fwd, up0)
    right /= np.linalg.norm(right)
    up = np.cross(right, fwd)
    f = 0.5 * min(width, height) / math.tan(half)
    near, far = dist - r, dist + r
    A, B = far / (far - near), -near * far / (far - near)
    # camera coordinates: xc = right.(X-eye), yc = up.(X-eye), zc = fwd.(X-eye) (> 0 in front)
    rows = [f * right + 0.5 * width * fwd, -f * up + 0.5 * height * fwd, A * fwd]
    offs = [-rows[0].dot(eye), -rows[1].dot(eye), -rows[2].dot(eye) + B]
    wrow = np.concatenate([fwd, [-fwd.dot(eye)]])
    out = np.concatenate([np.concatenate([rows[i], [offs[i]]]) for i in range(3)] + [wrow])
    return tuple(float(v) for v in out)


_AXES = {"x": (1.0, 0.0, 0.0), "y": (0.0, 1.0, 0.0), "z": (0.0, 0.0, 1.0)}
_VIEWS = {"+x": (0.0, 0.0), "-x": (180.0, 0.0), "+y": (90.0, 0.0), "-y": (-90.0, 0.0),
          "+z": (0.0, 90.0), "-z": (0.0, -90.0)}


def _parse_plane(text: str) -> Surface:
    t = text.strip()
    if "=" in t:
        ax, val = t.split("=", 1)
        ax = ax.strip().lower()
        if ax not in _AXES:
            raise ValueError(f"slice axis must be x, y or z, got {ax!r}")
        return Surface("slice", value=float(val), normal=_AXES[ax])
    parts = [float(v) for v in t.split(",")]
    if len(parts) != 4:
        raise ValueError(f"slice must be 'axis=c' or 'nx,ny,nz,c', got {text!r}")
    return Surface("slice", value=parts[3], normal=tuple(parts[:3]))


def pipeline_from_params(params: dict[str, str]) -> Pipeline:
    """Build a Pipeline from `<analysis type="insitu" .../>` attributes."""
    surfaces: list[Surface] = []
    for item in filter(None, (s.strip() for s in params.get("iso", "").split(";"))):
        if "=" not in item:
            raise ValueError(f"iso must be 'field=value', got {item!r}")
        name, val = item.rsplit("=", 1)
        surfaces.append(Surface("iso", field=name.strip(), value=float(val)))
    for item in filter(None, (s.strip() for s in params.get("slice", "").split(";"))):
        surfaces.append(_parse_plane(item))
    view = params.get("view", "+z").strip()
    if view in _VIEWS:
        vd = _VIEWS[view]
    else:
        a, e = view.split(",")
        vd = (float(a), float(e))
    return Pipeline(
        surfaces=tuple(surfaces),
        color_field=params.get("field", "velocity:mag"),
        width=int(params.get("width", 256)),
        height=int(params.get("height", 256)),
        view_dir=vd,
        vmin=float(params["vmin"]) if "vmin" in params else None,
        vmax=float(params["vmax"]) if "vmax" in params else None,
        composite=params.get("composite", "1") not in ("0", "false", "no"),
        continuous=params.get("continuous", "0") in ("1", "true", "yes"),
        projection=params.get("projection", "ortho"),
        fov=float(params.get("fov", 30.0)),
    )


@dataclass
class ExecuteResult:
    report: Report
    rgba: np.ndarray | None = None          # (H, W, 4) uint8 on the composite root
    depth: np.ndarray | None = None         # (H, W) float32
    view: tuple[float, ...] = field(default_factory=tuple)


class InsituAnalysis:
    """AnalysisAdaptor::Execute for a SemDataAdaptor (one per rank)."""

    def __init__(self, pipeline: Pipeline | dict[str, str]):
        self.pipeline = pipeline if isinstance(pipeline, Pipeline) else pipeline_from_params(pipeline)
        self._view: tuple[float, ...] | None = None
        self._native = None                 # (pipeline, view, NkbPipeline): marshalled once, reused per step
        self.executions = 0

    def view_for(self, data_adaptor) -> tuple[float, ...]:
        """The camera: fixed by the pipeline, or fitted once to the global
        mesh bounds on the first execute (nkb_mesh_bounds is collective, so
        every rank makes the same calls; reset_view() refits, on all ranks)."""
        p = self.pipeline
        if p.view is not None:
            return tuple(p.view)
        if self._view is None:
            b = data_adaptor.ctx.bounds()
            if p.projection == "perspective":
                self._view = perspective_view(b, p.width, p.height, *p.view_dir, fov=p.fov)
            elif p.projection == "ortho":
                self._view = ortho_view(b, p.width, p.height, *p.view_dir)
            else:
                raise ValueError(f"projection must be 'ortho' or 'perspective', got {p.projection!r}")
        return self._view

    def reset_view(self) -> None:
        self._view = None

    def execute(self, data_adaptor, fetch_image: bool = True, depth: bool = False) -> ExecuteResult:
        view = self.view_for(data_adaptor)
        ctx = data_adaptor.ctx
        if self._native is None or self._native[0] is not self.pipeline or self._native[1] != view:
            self._native = (self.pipeline, view, self.pipeline.native(view))
        rep = ctx.execute(self._native[2])
        self.executions += 1
        res = ExecuteResult(rep, view=view)
        root = (ctx.nranks == 1) or (not self.pipeline.composite) or ctx.rank == 0
        if fetch_image and root:
            if depth:
                res.rgba, res.depth = ctx.image(self.pipeline.width, self.pipeline.height, depth=True)
            else:
                res.rgba = ctx.image(self.pipeline.width, self.pipeline.height)
        return res

    def execute_async(self, data_adaptor) -> None:
        """Enqueue one step without waiting (nkb_execute_async): steps are
        ordered on the device only; `wait()` returns the last step's report."""
        view = self.view_for(data_adaptor)
        if self._native is None or self._native[0] is not self.pipeline or self._native[1] != view:
            self._native = (self.pipeline, view, self.pipeline.native(view))
        data_adaptor.ctx.execute_async(self._native[2])
        self._async_ctx = data_adaptor.ctx
        self.executions += 1

    def wait(self) -> Report:
        """Report of the last execute_async step (synchronises)."""
        return self._async_ctx.wait()

    def finalize(self) -> None:
        pass
