"""In situ hot-path benchmark: GLL points/s per in situ step
(adaptor + Q-criterion + isosurface/slice + render [+ composite]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...     (one rank per GPU)

A step = one AnalysisAdaptor::Execute over the rank's partition of the
workload, fields resident in HBM (`value`), plus the same step through the
reference-facing sink with host buffers (`e2e`).  Weak scaling: each GPU owns
one BASELINE configs[1] worth of elements (C2 RBC cylinder, 32,768 elements,
16.8M GLL points); at N GPUs the cylinder is N times taller.  `--impl
reference` times the CPU oracle port (the reference has no implementation of
this path) on all host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GLL points/sec per in situ step (adaptor+Q-crit+iso+render) at 1/2/4/8 B200"
UNIT = "GLL points/s"


class _StdoutToStderr:
    """Native libraries (NCCL's version banner) write to fd 1; the driver
    expects exactly one JSON line there.  Route fd 1 to fd 2 meanwhile."""

    def __enter__(self):
        sys.stdout.flush()
        self._saved = os.dup(1)
        os.dup2(2, 1)
        return self

    def __exit__(self, *exc):
        sys.stdout.flush()
        os.dup2(self._saved, 1)
        os.close(self._saved)
        return False


def _env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0}, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region (NVML in a
    thread every ~2 ms; falls back to nvidia-smi if NVML is unavailable)."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, device: int):
        self.device = device
        self.interval = float(os.environ.get("NKB_CLOCK_SAMPLE_MS", "2")) / 1e3   # NVML poll period
        self.samples: list[tuple[float, int]] = []
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        self._nv = None

    def start(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.device]) if vis else self.device
            self._h = nv.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
            self._nv = nv
        except Exception:
            self._nv = None
            return
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                mhz = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self.samples.append((float(mhz), int(rs)))
            except Exception:
                pass
            time.sleep(self.interval)

    def stop(self) -> dict:
        if self._nv is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"], "samples": 0}
        self._stop.set()
        self._t.join(timeout=2)
        nv = self._nv
        reasons = set()
        for _, rs in self.samples:
            for name, attr in self.REASONS:
                if hasattr(nv, attr) and rs & getattr(nv, attr):
                    reasons.add(name)
        sm = [m for m, _ in self.samples]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(sm)}


def _case_arrays(cfg: str, rank: int, world: int):
    from paper_2312_09888_b200 import synth

    return synth.make_case(cfg, rank, world, scale=world)


def _pipeline(case, width):
    from dataclasses import replace

    from paper_2312_09888_b200.analysis import pipeline_from_params

    p = pipeline_from_params({**case.params, "width": str(width), "height": str(width)})
    return replace(p, composite=True)


def _bytes_read_per_point(case, cached: bool = False, plane: bool | int = True) -> int:
    """Algorithmic HBM bytes the fused kernel reads per GLL point: every field
    component once (f64), the coordinates (`plane` True: all three unless the
    geometry cache replaces them; an int: the count of x,y,z the slice normals
    use, which is what K1g and K1s load), and the 9 cached
    Jacobian-inverse entries (72 B) when the cache is used."""
    b = 8 * sum(v.shape[0] for v in case.fields.values())
    if plane is not True and plane is not False:
        b += 8 * int(plane)
    elif not cached or plane:
        b += 24
    if cached:
        b += 72
    return b


WORKLOADS = {
    "c1": "c1: Taylor-Green box, 512 elements N=7",
    "c2": "c2: RBC cylinder, {E} elements N=7 ({N} x 32768; configs[1] per GPU)",
    "c3": "c3: turbPipe, {E} elements N=7 ({N} x 250000 along the pipe; configs[2] per GPU)",
    "c4": "c4: pebble bed, 1048576 elements N=7 (configs[3], partitioned over {N} GPUs)",
}


def run_ours(a):
    import numpy as np
    import torch

    from paper_2312_09888_b200.adaptor import SemDataAdaptor
    from paper_2312_09888_b200.analysis import InsituAnalysis
    from paper_2312_09888_b200.comm import Communicator
    from paper_2312_09888_b200.context import Context
    from paper_2312_09888_b200.data_model import POINT, FieldArray, SemBlock, Snapshot
    from paper_2312_09888_b200.device import DeviceArray, PinnedBuffer
    from paper_2312_09888_b200.sinks import InsituSink

    rank, world, local = _env_rank()
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("gloo")
    torch.cuda.set_device(local)
    with _StdoutToStderr():
        ctx = Context(local)
        comm = Communicator.from_torch(ctx) if world > 1 else None

    # the workload lives in HBM before timing starts (device-side generator)
    from paper_2312_09888_b200 import synth_device

    if a.config == "c1":
        hc = _case_arrays("c1", rank, world)
        dcase = synth_device.DeviceCase(hc.name, hc.n_elements, hc.e0, hc.n_elements_global,
                                        *(torch.from_numpy(v).cuda() for v in (hc.x, hc.y, hc.z)),
                                        {k: torch.from_numpy(v).cuda() for k, v in hc.fields.items()}, hc.params)
    else:
        dcase = synth_device.make_case(a.config, rank, world, scale=world, device=f"cuda:{local}")
    torch.cuda.synchronize()
    case = dcase
    npts = case.n_points
    pipe = _pipeline(case, a.width)
    fields = tuple(FieldArray(k, POINT, v.shape[0], v.reshape(-1), comp_stride=npts) for k, v in case.fields.items())
    blk = SemBlock(case.n_elements, case.x, case.y, case.z, fields=fields, element_offset=case.e0,
                   n_elements_global=case.n_elements_global)
    da = SemDataAdaptor(ctx)
    da.initialize(Snapshot(0.0, 0, rank, (blk,)))
    from dataclasses import replace

    # timed steps run without per-stage events (one-rank steps then replay a
    # captured CUDA graph); a second analysis with stage events gives the
    # per-kernel breakdown and the roofline's kernel time
    an = InsituAnalysis(pipe)
    an_t = InsituAnalysis(replace(pipe, timing=True))
    geo_build_ms = 0.0
    for _ in range(a.warmup):
        r = an_t.execute(da, fetch_image=False).report
        geo_build_ms = max(geo_build_ms, r.ms_geometry)
        an.execute(da, fetch_image=False)
    cached = bool(r.geometry_cached)
    plane = any(s.kind == "slice" for s in pipe.surfaces)
    if (plane and cached and r.surface_pass == 2) or r.surface_pass == 1:
        # K1g and K1s load only the coordinates with a nonzero normal component
        plane = sum(any(s.normal[c] != 0.0 for s in pipe.surfaces if s.kind == "slice") for c in range(3))
    bpp = _bytes_read_per_point(case, cached, plane)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    stream = torch.cuda.default_stream()
    clocks = ClockSampler(local)
    barrier()
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fused_ms, ntri, stages, surface_pass = [], 0, [], 0
    e0.record(stream)
    for _ in range(a.steps):
        res = an.execute(da, fetch_image=False)
    e1.record(stream)
    barrier()
    clk = clocks.stop()
    ms = max_over_ranks(e0.elapsed_time(e1)) / a.steps
    for _ in range(max(3, min(a.steps, 10))):          # stage breakdown (events around each stage)
        r = an_t.execute(da, fetch_image=False).report
        fused_ms.append(r.ms_fused)
        ntri = r.n_triangles
        surface_pass = r.surface_pass
        stages.append((r.ms_fused, r.ms_raster, r.ms_composite, r.ms_resolve))
    barrier()
    value = world * npts / (ms / 1e3)      # every rank holds npts (weak scaling)

    per_rank = [statistics.mean(fused_ms), float(ntri)]
    if dist is not None:
        gathered = [None] * world
        dist.all_gather_object(gathered, per_rank)
        per_rank_fused = [round(g[0], 4) for g in gathered]
        per_rank_tri = [int(g[1]) for g in gathered]
    else:
        per_rank_fused, per_rank_tri = [round(per_rank[0], 4)], [ntri]

    # roofline of the dominant kernel: the surface pass that ran -- K1g
    # (fused2_kernel: cached geometry, two CTAs per SM), K1 (fused_kernel) or,
    # without a velocity gradient, K1s (stream_kernel, warp per element)
    peaks, peak_kind = _peaks()
    fused = statistics.mean(fused_ms)
    alg_bytes = npts * bpp + 48 * ntri
    achieved = alg_bytes / (fused / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"traffic_{a.config}.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")

    # the same step without the geometry cache (x,y,z derivative pencils and
    # the cofactor/reciprocal chain recomputed every step), for comparison
    uncached = None
    if cached:
        ctx.set_geometry_cache(False)
        for _ in range(2):
            an_t.execute(da, fetch_image=False)
        um = [an_t.execute(da, fetch_image=False).report.ms_fused for _ in range(max(3, min(a.steps, 10)))]
        ctx.set_geometry_cache(True)
        an_t.execute(da, fetch_image=False)
        uncached = {"fused_ms": round(statistics.mean(um), 4),
                    "bytes_per_point": _bytes_read_per_point(case, False, plane)}

    # ---- end-to-end through the reference-facing sink with host buffers ----
    host_bytes = npts * _bytes_read_per_point(case, False, True)
    e2e = None
    hcase = None
    if host_bytes <= a.e2e_max_gb * 1e9:
        hcase = case.to_host()
        names = [("x", hcase.x), ("y", hcase.y), ("z", hcase.z)] + list(hcase.fields.items())
        pinned = PinnedBuffer(sum(v.nbytes for _, v in names))
        off, host = 0, {}
        for k, v in names:
            view = np.frombuffer((__import__("ctypes").c_byte * v.nbytes).from_address(pinned.ptr + off),
                                 dtype=np.float64)
            view[:] = v.ravel()
            view.setflags(write=False)          # immutable -> FieldArray aliases the pinned buffer
            host[k] = view.reshape(v.shape)
            off += v.nbytes
        hfields = tuple(FieldArray(k, POINT, hcase.fields[k].shape[0], host[k].ravel(), comp_stride=npts)
                        for k in hcase.fields)
        hblk = SemBlock(case.n_elements, host["x"], host["y"], host["z"], fields=hfields, element_offset=case.e0,
                        n_elements_global=case.n_elements_global)
        tmpdir = tempfile.mkdtemp(prefix="nkb_e2e_")
        # the PPM write of step i overlaps step i+1's H2D (writer thread); the
        # last write is waited for inside the timed region (sink.flush)
        params = {**case.params, "width": str(a.width), "height": str(a.width), "dir": tmpdir,
                  "async_write": "0" if a.e2e_sync_write else "1"}
        sink = InsituSink(params, comm=comm)
        e2e_steps = max(3, min(a.steps, 10))
        step = 0
        for _ in range(2):
            sink.consume(Snapshot(0.0, step, rank, (hblk,)))
            step += 1
        barrier()
        e0.record(stream)
        for _ in range(e2e_steps):
            sink.consume(Snapshot(0.0, step, rank, (hblk,)))
            step += 1
        sink.flush()
        e1.record(stream)
        barrier()
        e2e_ms = max_over_ranks(e0.elapsed_time(e1)) / e2e_steps
        sink.finalize()
        e2e = {"value": world * npts / (e2e_ms / 1e3), "unit": UNIT, "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": int(sink.adaptor.h2d_bytes), "d2h_bytes_per_step": int(a.width * a.width * 4 + 48),
               "path": "InsituSink.consume(host pinned snapshot) -> H2D -> execute -> D2H RGBA -> PPM"
                       + (" (written synchronously)" if a.e2e_sync_write else
                          " (written on a writer thread, overlapping the next step's H2D; last write waited for)")}
    else:
        e2e = {"value": None, "unit": UNIT, "h2d_bytes_per_step": int(host_bytes), "d2h_bytes_per_step": 0,
               "skipped": f"partition needs {host_bytes / 1e9:.1f} GB of pinned host memory (> --e2e-max-gb)"}

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded NekRS-layout SEM fields, synth.py)",
        "config": {
            "workload": WORKLOADS[a.config].format(E=case.n_elements_global, N=world),
            "elements_per_gpu": case.n_elements, "gll_points_per_gpu": npts,
            "gll_points_total": npts * world,
            **({"gll_points_unique": 185193} if a.config == "c1" else {}),
            "surfaces": case.params.get("iso", "") + (";slice " + case.params["slice"] if "slice" in case.params else ""),
            "color": case.params.get("field"), "image": f"{a.width}x{a.width}",
            "l2": f"inputs {npts * bpp / 1e9:.2f} GB/GPU >> 126 MB L2 (no flush needed)",
            "geometry_cache": ("on: d(r,s,t)/d(x,y,z) cached per mesh (static mesh), "
                               f"built once in {geo_build_ms:.3f} ms during warm-up") if cached else "off/not needed",
            "parallelism": f"element partition x{world}, sort-last depth composite"
                           + (" (P2P over NVLink peer memory unless NKB_COMPOSITE=nccl)" if world > 1 else ""),
        },
        "e2e": e2e,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                     "kernel": {1: "stream_kernel", 2: "fused2_kernel"}.get(surface_pass, "fused_kernel"),
                     "kernel_ms": fused, "alg_bytes_per_launch": alg_bytes, "peak_source": peak_kind,
                     "bytes_per_point": bpp, "triangles": ntri,
                     "frac_of_nominal_8tbs": achieved / 8000.0},
        "fused_uncached": uncached,
        "stages_ms": dict(zip(("fused", "raster", "composite", "resolve"),
                              (round(statistics.mean(x), 4) for x in zip(*stages)))),
        "fused_ms_per_rank": per_rank_fused,
        "triangles_per_rank": per_rank_tri,
        # libnekb200 kernels per step on rank 0: K1|K1s, zbuf clear, K2, range words, K3
        # (1 GPU or the NCCL composite, whose reduce kernels are NCCL's); the P2P
        # composite adds epoch, two waits, two signals and the composite kernel
        # and drops K3 (resolved inside the composite)
        "gpu_launches": (5 if world == 1 or os.environ.get("NKB_COMPOSITE") == "nccl" else 10) * a.steps,
        "clocks": clk,
    }
    if world == 1:
        out["next_rows"] = next_rows(ctx, da, case, hcase, peaks["hbm_gbs"], pipe)
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(hcase if hcase is not None else case.to_host(), pipe, an.view_for(da), a)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if comm is not None:
        comm.close()
    if dist is not None:
        dist.destroy_process_group()


def next_rows(ctx, da, case, hcase, hbm_gbs, pipe=None):
    """SURVEY.md §8f rows built after the hot path, measured on the same
    partition: the stats sink (nkb_stats, numpy-exact min/max/mean of every
    field) and the GPU checkpoint encoder (legacy-VTK sections).  Device
    time per call (synchronous ABI calls, wall clock around them) against the
    HBM roofline; numpy on the host copy of the same values beside it."""
    import time as _t

    import numpy as np

    from paper_2312_09888_b200.vtk import SemVtkWriter

    res = {}
    names = list(case.fields)
    segs = {n: [da.field_segment(n)] for n in names}
    nbytes = sum(8 * case.fields[n].shape[0] * case.n_points for n in names)
    for n in names:
        ctx.stats(segs[n])                                   # warm-up (plan + shapes)
    reps = 5
    t0 = _t.perf_counter()
    for _ in range(reps):
        got = {n: ctx.stats(segs[n]) for n in names}
    dt = (_t.perf_counter() - t0) / reps
    row = {"fields": names, "bytes": nbytes, "ms": dt * 1e3, "gb_per_s": nbytes / dt / 1e9,
           "frac_of_hbm": nbytes / dt / 1e9 / hbm_gbs}
    if hcase is not None:
        aos = {n: np.ascontiguousarray(hcase.fields[n].T).ravel() for n in names}
        t0 = _t.perf_counter()
        ref = {n: (v.min(), v.max(), v.mean()) for n, v in aos.items()}
        row["numpy_ms"] = (_t.perf_counter() - t0) * 1e3
        row["bit_exact_vs_numpy"] = all(
            np.array_equal(np.array(got[n]).view(np.uint64), np.array(ref[n]).view(np.uint64)) for n in names)
    res["stats_sink"] = row
    # DSSUM (continuous derived fields): setup once per mesh, then per field
    if case.name == "c2" and case.n_elements == 32768:
        import torch

        from paper_2312_09888_b200 import synth as _synth
        from paper_2312_09888_b200.analysis import InsituAnalysis as _IA

        gid = torch.from_numpy(_synth.lattice_ids((32, 32, 32), 0, 32768)).cuda()
        torch.cuda.synchronize()
        t0 = _t.perf_counter()
        ctx.mesh_set_global_ids(gid)
        setup = _t.perf_counter() - t0
        f = case.fields["temperature"].reshape(-1).clone()
        ctx.dssum(f)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            ctx.dssum(f)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        npts = case.n_points
        res["dssum"] = {"setup_ms": setup * 1e3, "ms": ms, "points": npts,
                        "gb_per_s_field": 16 * npts / ms / 1e6,
                        "note": "in-place average of one f64 field: read + write 8 B/pt, plus the sorted index"}
        # the whole continuous step (gradient pass -> DSSUM of Q -> surface pass)
        from dataclasses import replace as _rep

        if pipe is not None:
            ac, ad = _IA(_rep(pipe, continuous=True)), _IA(_rep(pipe, continuous=False))
            for a_ in (ac, ad):
                a_.execute(da, fetch_image=False)
            out = {}
            for key, a_ in (("continuous", ac), ("discontinuous", ad)):
                torch.cuda.synchronize()
                e0.record()
                for _ in range(reps):
                    a_.execute(da, fetch_image=False)
                e1.record()
                torch.cuda.synchronize()
                out[key] = e0.elapsed_time(e1) / reps
            res["dssum"]["step_ms"] = out
    w = SemVtkWriter(ctx)
    arrays = names + ["Q"]
    w.encode(da, arrays, 0, 0, 0.0)
    t0 = _t.perf_counter()
    data = w.encode(da, arrays, 0, 0, 0.0)
    dt = _t.perf_counter() - t0
    res["checkpoint_encode"] = {"arrays": arrays, "file_bytes": len(data), "ms": dt * 1e3,
                                "gb_per_s": len(data) / dt / 1e9,
                                "path": "GPU big-endian encode -> D2H into pinned host (file write not timed)"}
    return res


def _cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_baseline(case, pipe, view, a, reps: int = 2) -> dict:
    """CPU oracle port (oracle/sem_oracle.c), full step on all host cores."""
    from oracle import oracle as orc

    orc.build()
    cores = _cores()
    e_s = min(case.n_elements, 65536)              # bounded sample (~10-30 s of CPU work)
    sl = slice(0, e_s * 512)
    cf = orc.CaseFields(case.x[sl], case.y[sl], case.z[sl], {k: v[:, sl] for k, v in case.fields.items()})
    surf = [("iso", s.field, s.value) if s.kind == "iso" else ("slice", s.normal, s.value) for s in pipe.surfaces]
    best = math.inf
    for _ in range(reps):
        t0 = time.perf_counter()
        orc.pipeline_mt(cf, surf, pipe.color_field, view, pipe.width, pipe.height, cores)
        best = min(best, time.perf_counter() - t0)
    what = "full" if e_s == case.n_elements else f"first {e_s} of {case.n_elements} elements of the"
    return {"value": e_s * 512 / best, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{what} step (adaptor+Q+iso/slice+raster+resolve), best of {reps}, C oracle port, "
                      f"{cores} threads", "ms_per_step": best * 1e3}


def synth_elements(config: str, world: int) -> int:
    from paper_2312_09888_b200 import synth

    return synth.CONFIG_ELEMENTS[config] * (world if config in ("c2", "c3") else 1)


def run_reference(a):
    rank, world, _ = _env_rank()
    if rank != 0:
        return
    from oracle import oracle as orc
    from paper_2312_09888_b200.analysis import ortho_view

    orc.build()
    cores = _cores()
    case = _case_arrays(a.config, 0, 1)
    pipe = _pipeline(case, a.width)
    # bounded sample: first ~2 s worth of elements per step (measured rate ~1.3M pts/s/thread)
    e_sample = min(case.n_elements, max(64, int(2.0 * 1.3e6 * cores / 512)))
    sl = slice(0, e_sample * 512)
    cf = orc.CaseFields(case.x[sl], case.y[sl], case.z[sl], {k: v[:, sl] for k, v in case.fields.items()})
    b = (case.x.min(), case.x.max(), case.y.min(), case.y.max(), case.z.min(), case.z.max())
    view = ortho_view(b, pipe.width, pipe.height, *pipe.view_dir)
    surf = [("iso", s.field, s.value) if s.kind == "iso" else ("slice", s.normal, s.value) for s in pipe.surfaces]
    for _ in range(a.warmup):
        orc.pipeline_mt(cf, surf, pipe.color_field, view, pipe.width, pipe.height, cores)
    t0 = time.perf_counter()
    for _ in range(a.steps):
        orc.pipeline_mt(cf, surf, pipe.color_field, view, pipe.width, pipe.height, cores)
    dt = (time.perf_counter() - t0) / a.steps
    v = e_sample * 512 / dt
    sample = (f"{e_sample} of {case.n_elements} elements of {a.config} per step, full pipeline, "
              f"C oracle port on {cores} threads")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOADS[a.config].format(
                       E=synth_elements(a.config, world), N=world),
                   "image": f"{a.width}x{a.width}",
                   "cpu_sample": f"{e_sample} elements per step (bounded; throughput is per point)"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4"])
    ap.add_argument("--width", type=int, default=1024)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-max-gb", type=float, default=12.0)
    ap.add_argument("--e2e-sync-write", action="store_true", help="write each PPM inside consume() (no writer thread)")
    a = ap.parse_args()
    if a.warmup < 3:
        a.warmup = 3
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
