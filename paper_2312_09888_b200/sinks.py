"""Analysis sinks (the AnalysisAdaptors the bridge drives), GPU-backed.

Same plugin contract as the reference (pkg/src/nekmini/sinks.py:310-418):
``cls(params: dict[str, str])`` creates its output directory and fails fast
when it is unwritable (:396-402), ``consume(snapshot) -> int`` returns the
bytes written, ``finalize()`` flushes.  Registered kinds:

* ``render`` -- drop-in for the reference's RenderSink (:327-351): the 2D
  pseudocolor of a structured snapshot, computed by libnekb200
  (nkb_render_structured) and byte-identical to the reference's `render`
  (:245-295); same default two images (temperature, velocity:mag), same
  file names ``step{step:06d}_{field with ':'->'_'}.ppm``.
* ``insitu`` -- the SEM hot path: adaptor -> Q -> iso/slice -> raster ->
  composite (analysis.InsituAnalysis); writes one PPM per trigger on the
  composite root.
* ``stats`` -- drop-in for the reference's StatsSink (:366-393): appends
  ``step,time,field,min,max,mean`` rows; the reductions run on the GPU
  (nkb_stats) with numpy's exact arithmetic, so the rows are byte-identical.
* ``checkpoint`` -- legacy-VTK checkpoints (:310-324): structured snapshots
  in the reference's exact STRUCTURED_POINTS layout; SEM snapshots as an
  UNSTRUCTURED_GRID of the sub-hex mesh with the snapshot's fields plus any
  AddArray arrays (``arrays="Q,vorticity:mag"``), encoded on the GPU (vtk.py).
* ``transit`` -- the in transit mode: SEM partitions staged GPU-to-GPU to
  an endpoint rank (NCCL), analysed there on the assembled mesh.
* ``null`` -- counts invocations (:354-363).
"""
from __future__ import annotations

from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _native as N
from .adaptor import SemDataAdaptor
from .analysis import InsituAnalysis, pipeline_from_params
from .context import Context
from .data_model import CELL, SemBlock, check_assembly
from .device import DeviceArray, device_ptr, is_device_array


@dataclass(frozen=True)
class ColorMap:
    """Piecewise-linear RGB colormap over t in [0, 1] (sinks.py:190-209)."""

    anchors: tuple[tuple[float, tuple[int, int, int]], ...]

    def __post_init__(self):
        ts = [t for t, _ in self.anchors]
        if ts[0] != 0.0 or ts[-1] != 1.0 or any(b <= a for a, b in zip(ts, ts[1:])):
            raise ValueError("anchor positions must strictly increase from 0 to 1")


DEFAULT_COLORMAP = ColorMap(((0.0, (59, 76, 192)), (0.5, (255, 255, 255)), (1.0, (180, 4, 38))))


@dataclass(frozen=True)
class ImageRGB:
    width: int
    height: int
    pixels: bytes  # row-major 8-bit RGB, top row first

    def __post_init__(self):
        if len(self.pixels) != 3 * self.width * self.height:
            raise ValueError("pixel buffer length must be 3 * width * height")


def write_ppm(img: ImageRGB, path) -> int:
    """Binary PPM (P6); returns the exact byte count written (sinks.py:298-303)."""
    header = f"P6\n{img.width} {img.height}\n255\n".encode("ascii")
    data = header + img.pixels
    Path(path).write_bytes(data)
    return len(data)


def _probe_writable(d: Path):
    probe = d / ".write_probe"
    try:
        probe.touch()
        probe.unlink()
    except OSError as e:
        raise OSError(f"output directory {d} is not writable: {e}") from e


_CTX: dict[int, Context] = {}


def default_context(device: int | None = None) -> Context:
    """One libnekb200 context per (process, device)."""
    if device is None:
        import os
        device = int(os.environ.get("LOCAL_RANK", "0"))
    if device not in _CTX:
        _CTX[device] = Context(device)
    return _CTX[device]


class GpuRenderer:
    """GPU implementation of the reference's `render` (sinks.py:245-295)."""

    def __init__(self, ctx: Context | None = None):
        self._ctx = ctx
        self._staging: dict[tuple[int, str], DeviceArray] = {}
        self._rgb: DeviceArray | None = None

    @property
    def ctx(self) -> Context:
        if self._ctx is None:        # created on first use: constructing a sink needs no GPU
            self._ctx = default_context()
        return self._ctx

    def render(self, s, field: str, cmap: ColorMap = DEFAULT_COLORMAP, width: int = 256, height: int = 256,
               vmin: float | None = None, vmax: float | None = None) -> ImageRGB:
        if cmap != DEFAULT_COLORMAP:
            raise ValueError("the GPU renderer implements the reference DEFAULT_COLORMAP only")
        blocks = list(s.blocks)
        if not blocks:
            raise ValueError("no blocks to assemble")
        check_assembly(blocks)
        base, _, derived = field.partition(":")
        f0 = blocks[0].field_named(base)
        if f0.association == CELL and len(blocks) == 1:
            raise ValueError("cell fields cannot be rendered as a point grid")
        comps = f0.components
        if derived == "":
            if comps != 1:
                raise ValueError(
                    f"field {base!r} has {comps} components; request a derived scalar such as {base!r}:mag"
                )
            mode = 0
        elif derived == "mag":
            mode = 1
        else:
            raise ValueError(f"unknown derived scalar {derived!r}")
        ni0, nj, nk = blocks[0].dims
        dev_blocks = []
        for bi, b in enumerate(blocks):
            vals = b.field_named(base).values
            if is_device_array(vals):
                d = vals
            else:
                a = np.ascontiguousarray(vals, dtype=np.float64)
                key = (bi, base)
                d = self._staging.get(key)
                if d is None or d.size != a.size:
                    d = DeviceArray.empty(self.ctx, (a.size,), np.float64)
                    self._staging[key] = d
                d.upload(a, sync=False)
            dev_blocks.append((d, b.dims[0]))
        npx = width * height * 3
        if self._rgb is None or self._rgb.size < npx:
            self._rgb = DeviceArray.empty(self.ctx, (npx,), np.uint8)
        nan = float("nan")
        self.ctx.render_structured(
            dev_blocks, nj * nk, comps, mode, width, height,
            nan if vmin is None else float(vmin), nan if vmax is None else float(vmax), self._rgb,
        )
        out = np.empty(npx, np.uint8)
        N.call("nkb_memcpy", out.ctypes.data, self._rgb.ptr, npx, 2, None)
        N.call("nkb_stream_sync", None)
        return ImageRGB(width, height, out.tobytes())


_RENDERER: GpuRenderer | None = None


def render(s, field: str, cmap: ColorMap = DEFAULT_COLORMAP, width: int = 256, height: int = 256,
           vmin: float | None = None, vmax: float | None = None) -> ImageRGB:
    """Drop-in for the reference `render` (sinks.py:245-295), on the GPU."""
    global _RENDERER
    if _RENDERER is None:
        _RENDERER = GpuRenderer()
    return _RENDERER.render(s, field, cmap, width, height, vmin, vmax)


class RenderSink:
    """Renders per trigger; with no explicit field, renders two images
    (temperature and velocity magnitude) per snapshot (sinks.py:327-351)."""

    def __init__(self, params: dict[str, str], comm=None):
        self.dir = Path(params.get("dir", "render_out"))
        self.width = int(params.get("width", 256))
        self.height = int(params.get("height", 256))
        f = params.get("field")
        self.fields = [f] if f else ["temperature", "velocity:mag"]
        self.vmin = float(params["vmin"]) if "vmin" in params else None
        self.vmax = float(params["vmax"]) if "vmax" in params else None
        self.dir.mkdir(parents=True, exist_ok=True)
        _probe_writable(self.dir)
        self._renderer = GpuRenderer()

    def consume(self, s) -> int:
        total = 0
        for name in self.fields:
            img = self._renderer.render(s, name, DEFAULT_COLORMAP, self.width, self.height, self.vmin, self.vmax)
            fname = f"step{s.step:06d}_{name.replace(':', '_')}.ppm"
            total += write_ppm(img, self.dir / fname)
        return total

    def finalize(self):
        pass


class InsituSink:
    """The SEM in situ analysis as a sink: one image per trigger on the
    composite root, named like the reference's render images (sinks.py:346)."""

    def __init__(self, params: dict[str, str], comm=None):
        self.dir = Path(params.get("dir", "insitu_out"))
        self.pipeline = pipeline_from_params(params)
        self.comm = comm
        self.velocity = params.get("velocity", "velocity")
        self.adaptor: SemDataAdaptor | None = None   # created on first consume (needs the GPU)
        self.analysis = InsituAnalysis(self.pipeline)
        self.last = None
        # async_write=1: the PPM write of step i runs on a writer thread while
        # step i+1's fields cross PCIe; consume() waits for the previous write
        # before the library's pinned PPM buffer is reused, and flush() /
        # finalize() wait for the last one.  Default 0: the file is complete
        # when consume() returns, as in the reference (sinks.py:346-351).
        self.async_write = params.get("async_write", "0").strip().lower() in ("1", "true", "yes", "on")
        self._writer = None
        self._pending = None
        # who writes: the composite root, or -- composite="0" on several
        # ranks -- every rank, its own partial image under a rank-suffixed name
        self.per_rank = comm is not None and comm.size > 1 and not self.pipeline.composite
        if comm is None or comm.rank == 0 or self.per_rank:
            self.dir.mkdir(parents=True, exist_ok=True)
            _probe_writable(self.dir)

    def consume(self, s) -> int:
        if self.adaptor is None:
            ctx = self.comm.ctx if self.comm is not None else default_context()
            self.adaptor = SemDataAdaptor(ctx, velocity=self.velocity)
        self.adaptor.initialize(s)
        ctx = self.adaptor.ctx
        res = self.analysis.execute(self.adaptor, fetch_image=False)
        self.last = res
        if not ((ctx.nranks == 1) or (not self.pipeline.composite) or ctx.rank == 0):
            return 0
        self.flush()                  # the previous write still reads the pinned PPM buffer
        # header + RGB packed on the GPU into pinned memory: same bytes as
        # write_ppm(ImageRGB(w, h, rgba[..., :3].tobytes())) (sinks.py:298-303)
        ppm = ctx.image_ppm()
        suffix = f"_rank{ctx.rank:04d}" if self.per_rank else ""
        path = self.dir / f"step{s.step:06d}_{self.pipeline.color_field.replace(':', '_')}{suffix}.ppm"
        if self.async_write:
            if self._writer is None:
                from concurrent.futures import ThreadPoolExecutor

                self._writer = ThreadPoolExecutor(max_workers=1, thread_name_prefix="nkb-ppm")
            # the write reads the context's pinned PPM buffer: every later
            # image_ppm on this context (any sink) waits for it first
            self._pending = self._writer.submit(_write_bytes, path, ppm)
            ctx.hold_ppm(self._pending)
        else:
            _write_bytes(path, ppm)
        return len(ppm)

    def flush(self):
        """Wait for the pending PPM write (async_write); re-raises its error."""
        pending, self._pending = self._pending, None
        if pending is not None:
            pending.result()

    def finalize(self):
        try:
            self.flush()
        finally:
            if self._writer is not None:
                self._writer.shutdown(wait=True)
                self._writer = None


def _write_bytes(path, data) -> None:
    with open(path, "wb") as f:
        f.write(data)


def _device_len(d) -> int:
    shape = d.__cuda_array_interface__["shape"]
    return int(np.prod(shape)) if len(shape) else 1


class TransitSink:
    """In transit analysis (the paper's staging mode; reference transport.py
    N:1 endpoint, :358-376): every rank's SEM partition is staged to the
    endpoint GPU over NCCL send/recv (nkb_transit_gather, no host copy), and
    the endpoint runs the in situ pipeline on the assembled mesh alone and
    writes the image.  Same attributes as ``insitu`` plus ``endpoint``."""

    def __init__(self, params: dict[str, str], comm=None):
        from dataclasses import replace

        self.dir = Path(params.get("dir", "transit_out"))
        self.pipeline = replace(pipeline_from_params(params), composite=False)
        self.endpoint = int(params.get("endpoint", 0))
        self.comm = comm
        self.velocity = params.get("velocity", "velocity")
        self.analysis = InsituAnalysis(self.pipeline)
        self.adaptor: SemDataAdaptor | None = None
        self.last = None
        if comm is None or comm.rank == self.endpoint:
            self.dir.mkdir(parents=True, exist_ok=True)
            _probe_writable(self.dir)

    def consume(self, s) -> int:
        if self.adaptor is None:
            ctx = self.comm.ctx if self.comm is not None else default_context()
            self.adaptor = SemDataAdaptor(ctx, velocity=self.velocity)
            if self.comm is not None and self.comm.rank == self.endpoint:
                # the endpoint alternates between its partition and the
                # assembled mesh: recomputing J^-1 is cheaper than re-caching it
                ctx.set_geometry_cache(False)
        self.adaptor.initialize(s)
        ctx = self.adaptor.ctx
        view = self.analysis.view_for(self.adaptor)            # collective (global bounds)
        if self.comm is not None and ctx.nranks > 1:
            ctx.transit_gather(self.endpoint)
            if ctx.rank != self.endpoint:
                return 0
        self.last = ctx.execute(self.pipeline.native(view))
        ppm = ctx.image_ppm()
        fname = f"step{s.step:06d}_{self.pipeline.color_field.replace(':', '_')}.ppm"
        with open(self.dir / fname, "wb") as f:
            f.write(ppm)
        return len(ppm)

    def finalize(self):
        pass


class StatsSink:
    """Appends step,time,field,min,max,mean rows (sinks.py:366-393).

    Structured snapshots (the reference's data model): every block, point and
    component of each field, concatenated in block order, exactly as
    ``np.concatenate([b.field_named(name).values for b in s.blocks])``.  SEM
    snapshots: the rank's SemBlock; with a communicator the statistics are
    global (all ranks' values in rank order) and rank 0 writes the file.
    min / max / mean come from nkb_stats, bit-identical to numpy's."""

    HEADER = "step,time,field,min,max,mean"

    def __init__(self, params: dict[str, str], comm=None):
        self.path = Path(params["path"])
        self.comm = comm
        self.root = comm is None or comm.rank == 0
        if self.root:
            if self.path.parent != Path(""):
                self.path.parent.mkdir(parents=True, exist_ok=True)
            if not self.path.exists():
                self.path.write_text(self.HEADER + "\n")
            _probe_writable(self.path.parent)
        self._ctx: Context | None = None
        self._adaptor: SemDataAdaptor | None = None
        self._staging: dict[tuple[int, str], DeviceArray] = {}

    @property
    def ctx(self) -> Context:
        if self._ctx is None:
            self._ctx = self.comm.ctx if self.comm is not None else default_context()
        return self._ctx

    def _segments(self, s) -> tuple[list[str], dict[str, list], bool]:
        blocks = list(s.blocks)
        names = [f.name for f in blocks[0].fields]
        if isinstance(blocks[0], SemBlock):
            if self._adaptor is None:
                self._adaptor = SemDataAdaptor(self.ctx)
            self._adaptor.initialize(s)
            return names, {n: [self._adaptor.field_segment(n)] for n in names}, self.comm is not None
        segs: dict[str, list] = {}
        for name in names:
            lst = []
            for bi, b in enumerate(blocks):
                vals = b.field_named(name).values
                if is_device_array(vals):
                    d = vals
                else:
                    a = np.ascontiguousarray(vals, dtype=np.float64).ravel()
                    d = self._staging.get((bi, name))
                    if d is None or d.size != a.size:
                        d = DeviceArray.empty(self.ctx, (a.size,), np.float64)
                        self._staging[(bi, name)] = d
                    d.upload(a, sync=False)
                n = _device_len(d)
                lst.append((device_ptr(d), n, 1, n))
            segs[name] = lst
        return names, segs, False

    def consume(self, s) -> int:
        names, segs, collective = self._segments(s)
        rows = []
        for name in names:
            mn, mx, mean = self.ctx.stats(segs[name], collective)
            rows.append(f"{s.step},{s.time:.17g},{name},{mn:.17g},{mx:.17g},{mean:.17g}")
        text = "\n".join(rows) + "\n"
        if not self.root:
            return 0
        with open(self.path, "a") as f:
            f.write(text)
        return len(text)

    def finalize(self):
        pass


class CheckpointSink:
    """One legacy-VTK file per block and trigger (sinks.py:310-324)."""

    def __init__(self, params: dict[str, str], comm=None):
        self.dir = Path(params.get("dir", "checkpoint_out"))
        self.format = params.get("format", "binary")
        if self.format not in ("ascii", "binary"):
            raise ValueError(f"checkpoint format must be ascii or binary, got {self.format!r}")
        self.extra = [a.strip() for a in params.get("arrays", "").split(",") if a.strip()]
        self.comm = comm
        self.dir.mkdir(parents=True, exist_ok=True)
        _probe_writable(self.dir)
        self._adaptor: SemDataAdaptor | None = None
        self._writer = None

    def consume(self, s) -> int:
        from .vtk import SemVtkWriter, checkpoint_filename, checkpoint_write

        blocks = list(s.blocks)
        if not (blocks and isinstance(blocks[0], SemBlock)):
            _, total = checkpoint_write(s, self.dir, self.format)
            return total
        if self.format != "binary":
            raise ValueError("SEM checkpoints are written in binary only")
        if self._adaptor is None:
            ctx = self.comm.ctx if self.comm is not None else default_context()
            self._adaptor = SemDataAdaptor(ctx)
            self._writer = SemVtkWriter(ctx)
        self._adaptor.initialize(s)
        arrays = list(dict.fromkeys([f.name for f in blocks[0].fields] + self.extra))
        data = self._writer.encode(self._adaptor, arrays, s.step, s.producer_id, s.time)
        with open(self.dir / checkpoint_filename(s.step, s.producer_id), "wb") as f:
            f.write(data)
        return len(data)

    def finalize(self):
        pass


class NullSink:
    def __init__(self, params: dict[str, str] | None = None, comm=None):
        self.count = 0

    def consume(self, s) -> int:
        self.count += 1
        return 0

    def finalize(self):
        pass


_SINK_TYPES = {
    "render": RenderSink,
    "insitu": InsituSink,
    "transit": TransitSink,
    "stats": StatsSink,
    "checkpoint": CheckpointSink,
    "null": NullSink,
}


def make_sink(kind: str, params: dict[str, str], comm=None):
    try:
        cls = _SINK_TYPES[kind]
    except KeyError:
        raise ValueError(f"unknown sink kind {kind!r}") from None
    return cls(params, comm=comm)
