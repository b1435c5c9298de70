"""In situ hot-path benchmark: GLL points/s per in situ step
(adaptor + Q-criterion + isosurface/slice + render [+ composite]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...     (one rank per GPU)

`python bench.py --gpus N` without torchrun spawns its own N ranks (the
reference harness spawns its producers the same way, harness.py:222-275);
under torchrun WORLD_SIZE must equal N.

A step = one AnalysisAdaptor::Execute over the rank's partition of the
workload, fields resident in HBM (`value`), plus the same step through the
reference-facing sink with host buffers (`e2e`).  Configs (BASELINE.json
`configs`):
  c2 (default)  RBC cylinder, 32,768 elements per GPU (weak: the cylinder is N
                times taller at N GPUs)
  c1            Taylor-Green box, 512 elements
  c3            turbPipe; --scaling weak (250,000 elements per GPU, default)
                or strong (250,000 elements split over the N GPUs)
  c4            pebble bed, 1,048,576 elements split over the N GPUs
  c5            weak-scaling box, --elements E (65,536 .. 2,097,152) split
                over the N GPUs (default E = 65,536 x N: the 64K-per-GPU diagonal)
c1/c2 inputs come from the numpy generator (synth.py) so the reference arm
consumes the identical bytes; c3-c5 are generated on the device
(synth_device.py).  `--impl reference` times the CPU oracle port (the
reference has no implementation of this path) on all host cores.
"""
from __future__ import annotations

import argparse
import csv
import hashlib
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GLL points/sec per in situ step (adaptor+Q-crit+iso+render) at 1/2/4/8 B200"
UNIT = "GLL points/s"
NN = 512
# reference timings.csv schema (reporting.py:21), plus the roofline columns
TIMINGS_HEADER = ["label", "step", "phase", "seconds"]
PHASES_HEADER = TIMINGS_HEADER + ["gll_points", "alg_bytes", "roofline_frac"]


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


def _cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region (NVML in a
    thread every ~2 ms)."""

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


# ---------------------------------------------------------------------------
# workload description: shared by both arms so their `config` dicts match
# ---------------------------------------------------------------------------

class Workload:
    """Global element count, per-rank partition and scaling mode of a run."""

    def __init__(self, a, world: int):
        from paper_2312_09888_b200 import synth

        self.config = a.config
        if a.config in ("c2", "c3") and a.scaling == "weak":
            self.scale, self.scaling = world, "weak"
        elif a.config == "c5":
            self.scale = int(a.elements) if a.elements else 65536 * world
            self.scaling = "weak" if self.scale == 65536 * world else "strong"
        else:
            self.scale, self.scaling = 1, ("weak" if world == 1 else "strong")
        self.world = world
        self.n_global = synth.global_elements(a.config, self.scale)
        self.max_per_rank = max(synth.partition(self.n_global, r, world)[1] - synth.partition(self.n_global, r, world)[0]
                                for r in range(world))
        self.params = dict(synth.PARAMS[a.config])
        self.host_generated = a.config in ("c1", "c2")

    def describe(self) -> str:
        E, N = self.n_global, self.world
        if self.config == "c1":
            return "c1: Taylor-Green box, 512 elements N=7 (configs[0])"
        if self.config == "c2":
            return f"c2: RBC cylinder, {E} elements N=7 ({N} x 32768; configs[1] per GPU)"
        if self.config == "c3":
            if self.scaling == "weak":
                return f"c3: turbPipe, {E} elements N=7 ({N} x 250000 along the pipe; configs[2] per GPU)"
            return f"c3: turbPipe, {E} elements N=7 (configs[2], strong: partitioned over {N} GPUs)"
        if self.config == "c4":
            return f"c4: pebble bed, {E} elements N=7 (configs[3], partitioned over {N} GPUs)"
        return f"c5: weak-scaling box, {E} elements N=7 ({E // N} per GPU x {N}; configs[4])"


def _surfaces_text(params) -> str:
    return params.get("iso", "") + (";slice " + params["slice"] if "slice" in params else "")


def _pipeline(params, width):
    from dataclasses import replace

    from paper_2312_09888_b200.analysis import pipeline_from_params

    p = pipeline_from_params({**params, "width": str(width), "height": str(width)})
    return replace(p, composite=True)


def pipeline_bytes(pipe, comps: dict) -> dict:
    """SURVEY.md §8(d) algorithmic HBM bytes per GLL point of one step: every
    field component the pipeline reads (f64), plus the coordinates: all three
    when a velocity gradient is needed (the Jacobian), else the ones a slice
    normal uses.  Caches of derived geometry are NOT algorithmic bytes."""
    names = [s.field for s in pipe.surfaces if s.kind == "iso"] + [pipe.color_field]
    need_grad = any(n in ("Q", "vorticity", "vorticity:mag") for n in names)
    read = {"velocity"} if need_grad else set()
    for n in names:
        if n.endswith(":mag") and n != "vorticity:mag":
            read.add(n[:-4])
        elif n in comps:
            read.add(n)
    field_b = 8 * sum(comps[n] for n in read if n in comps)
    axes = sum(any(s.kind == "slice" and s.normal[c] != 0.0 for s in pipe.surfaces) for c in range(3))
    coord_b = 24 if need_grad else 8 * axes
    return {"alg": field_b + coord_b, "fields": field_b, "plane_axes": axes, "need_grad": need_grad}


def common_config(wl: Workload, a) -> dict:
    """The `config` object both arms print (identical keys and values)."""
    from paper_2312_09888_b200 import synth

    comps = {"velocity": 3, "temperature": 1}
    pb = pipeline_bytes(_pipeline(wl.params, a.width), comps)
    per_rank_bytes = wl.max_per_rank * NN * pb["alg"]
    return {
        "workload": wl.describe(),
        "elements_total": wl.n_global,
        "elements_per_gpu": wl.max_per_rank,
        "gll_points_total": wl.n_global * NN,
        "gll_points_per_gpu": wl.max_per_rank * NN,
        **({"gll_points_unique": 185193} if wl.config == "c1" else {}),
        "surfaces": _surfaces_text(wl.params),
        "color": wl.params.get("field"),
        "image": f"{a.width}x{a.width}",
        "scaling_mode": wl.scaling,
        "l2": (f"inputs {per_rank_bytes / 1e9:.2f} GB/GPU >> 126 MB L2 (no flush needed)" if per_rank_bytes > 5e8
               else f"inputs {per_rank_bytes / 1e6:.1f} MB/GPU: L2-resident, not flushed (latency case)"),
        "inputs": "numpy generator (synth.py), identical bytes in both arms" if wl.host_generated
                  else "device generator (synth_device.py)",
        "parallelism": f"element partition x{wl.world}, sort-last depth composite",
    }


def _digest(arrays) -> str:
    h = hashlib.blake2b(digest_size=16)
    for v in arrays:
        h.update(memoryview(v).cast("B"))
    return h.hexdigest()


def _case_digest(hcase) -> str:
    import numpy as np

    return _digest([np.ascontiguousarray(v) for v in (hcase.x, hcase.y, hcase.z)]
                   + [np.ascontiguousarray(hcase.fields[k]) for k in sorted(hcase.fields)])


def _fp64_peak():
    """Measured DFMA peak of this GPU (tools/fp64_probe.cu); TF/s or None."""
    import ctypes

    so = os.path.join(ROOT, "paper_2312_09888_b200", "lib", "libnkbprobe.so")
    try:
        L = ctypes.CDLL(so)
    except OSError:
        return None
    best, med = ctypes.c_double(), ctypes.c_double()
    if L.nkb_probe_fp64(ctypes.byref(best), ctypes.byref(med), 10) != 0:
        return None
    return {"tflops": best.value, "tflops_median": med.value,
            "how": "tools/fp64_probe.cu: 8 independent DFMA chains x 4096 per thread, 8 CTAs x 256 threads "
                   "per SM, best of 10 (CUDA events)"}


def _profile_json(name):
    p = os.path.join(ROOT, "profiles", name)
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return None


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def _make_cases(wl: Workload, rank: int, world: int, local: int):
    """(device case, host case or None) for this rank's partition."""
    import torch

    from paper_2312_09888_b200 import synth, synth_device

    if wl.host_generated:
        hc = synth.make_case(wl.config, rank, world, scale=wl.scale)
        dc = synth_device.DeviceCase(hc.name, hc.n_elements, hc.e0, hc.n_elements_global,
                                     *(torch.from_numpy(v).to(f"cuda:{local}") for v in (hc.x, hc.y, hc.z)),
                                     {k: torch.from_numpy(v).to(f"cuda:{local}") for k, v in hc.fields.items()},
                                     hc.params)
        return dc, hc
    dc = synth_device.make_case(wl.config, rank, world, scale=wl.scale, device=f"cuda:{local}")
    return dc, None


WORK_TRI_WEIGHT = 0.021   # K1s: one triangle costs 0.021 element passes (C4, 4 ranks: per-rank time = a E + b T)


def _work_cuts(ctx, case, rank, world, dist, width):
    """Contiguous element ranges of equal surface-pass cost (--partition work):
    one ordered step on the equal partition gives every element's triangle
    count, the ranks all-gather them, and the cuts split the prefix sum of
    1 + WORK_TRI_WEIGHT x triangles into equal parts (what a solver's
    partitioner does with element weights; the step itself is untimed)."""
    import numpy as np

    from dataclasses import replace

    from paper_2312_09888_b200.analysis import InsituAnalysis

    pipe = _pipeline(case.params, width)
    da = _sem_adaptor(ctx, case, rank)
    InsituAnalysis(replace(pipe, emit_meta=True, composite=False)).execute(da, fetch_image=False)
    _, meta = ctx.triangles(with_meta=True)
    tris = np.bincount((np.asarray(meta) >> np.uint64(32)).astype(np.int64), minlength=case.n_elements)
    parts = [None] * world
    dist.all_gather_object(parts, (case.e0, tris[:case.n_elements]))
    tri_g = np.concatenate([t for _, t in sorted(parts, key=lambda p: p[0])])
    del da
    return balanced_cuts(tri_g, world)


def balanced_cuts(tri_per_element, world, weight=None):
    """world + 1 element indices: contiguous ranges whose costs 1 + weight x
    triangles per element are as equal as the element granularity allows
    (every range non-empty when there are at least `world` elements)."""
    import numpy as np

    w = WORK_TRI_WEIGHT if weight is None else weight
    cs = np.cumsum(1.0 + w * np.asarray(tri_per_element, dtype=np.float64))
    n = len(cs)
    cuts = [0] + [int(np.searchsorted(cs, cs[-1] * k / world)) + 1 for k in range(1, world)] + [n]
    for k in range(1, world):                          # increasing, room for the ranks after k
        cuts[k] = min(max(cuts[k], cuts[k - 1] + 1), n - (world - k))
    return cuts


def _host_sample(dcase, e_s: int):
    """Host copy of the first e_s elements of a device case (the oracle's input)."""
    from paper_2312_09888_b200 import synth

    n = e_s * NN
    return synth.SemCase(dcase.name, e_s, dcase.e0, dcase.n_elements_global,
                         dcase.x[:n].cpu().numpy(), dcase.y[:n].cpu().numpy(), dcase.z[:n].cpu().numpy(),
                         {k: v[:, :n].contiguous().cpu().numpy() for k, v in dcase.fields.items()},
                         dict(dcase.params))


def _sem_adaptor(ctx, dcase, rank, n_elements=None):
    from paper_2312_09888_b200.adaptor import SemDataAdaptor
    from paper_2312_09888_b200.data_model import POINT, FieldArray, SemBlock, Snapshot

    E = dcase.n_elements if n_elements is None else n_elements
    n = E * NN
    if E == dcase.n_elements:
        xs, ys, zs = dcase.x, dcase.y, dcase.z
        fl = {k: v.reshape(-1) for k, v in dcase.fields.items()}
        stride = dcase.n_points
    else:
        xs, ys, zs = dcase.x[:n].contiguous(), dcase.y[:n].contiguous(), dcase.z[:n].contiguous()
        fl = {k: v[:, :n].contiguous().reshape(-1) for k, v in dcase.fields.items()}
        stride = n
    fields = tuple(FieldArray(k, POINT, dcase.fields[k].shape[0], v, comp_stride=stride) for k, v in fl.items())
    blk = SemBlock(E, xs, ys, zs, fields=fields, element_offset=dcase.e0,
                   n_elements_global=dcase.n_elements_global if n_elements is None else E)
    da = SemDataAdaptor(ctx)
    da.initialize(Snapshot(0.0, 0, rank, (blk,)))
    da._keep = (xs, ys, zs, fl)
    return da


def run_ours(a):
    import numpy as np
    import torch

    from paper_2312_09888_b200.analysis import InsituAnalysis
    from paper_2312_09888_b200.comm import Communicator
    from paper_2312_09888_b200.context import Context
    from paper_2312_09888_b200.data_model import POINT, FieldArray, SemBlock, Snapshot
    from paper_2312_09888_b200.device import PinnedBuffer
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
    wl = Workload(a, world)
    config = common_config(wl, a)

    # the workload lives in HBM before timing starts
    case, hcase = _make_cases(wl, rank, world, local)
    torch.cuda.synchronize()
    cuts = None
    if a.partition == "work" and world > 1 and not wl.host_generated:
        from paper_2312_09888_b200 import synth_device

        cuts = _work_cuts(ctx, case, rank, world, dist, a.width)
        del case
        torch.cuda.empty_cache()
        case = synth_device.make_case(wl.config, rank, world, scale=wl.scale, device=f"cuda:{local}", cuts=cuts)
        torch.cuda.synchronize()
        config["partition"] = {"kind": "contiguous element ranges balancing the surface-pass cost",
                               "cost_per_element": f"1 + {WORK_TRI_WEIGHT} x triangles (K1s cost model, C4)",
                               "cuts": [int(c) for c in cuts]}
    npts = case.n_points
    pipe = _pipeline(case.params, a.width)
    comps = {k: v.shape[0] for k, v in case.fields.items()}
    pb = pipeline_bytes(pipe, comps)
    da = _sem_adaptor(ctx, case, rank)
    from dataclasses import replace

    # timed steps run without per-stage events (steps replay a captured CUDA
    # graph); a second analysis with stage events gives the per-kernel
    # breakdown and the roofline's kernel time
    an = InsituAnalysis(pipe)
    an_t = InsituAnalysis(replace(pipe, timing=True))
    geo_build_ms = 0.0
    for _ in range(a.warmup):
        r = an_t.execute(da, fetch_image=False).report
        geo_build_ms = max(geo_build_ms, r.ms_geometry)
        an.execute(da, fetch_image=False)
    # the stream-ordered steps capture their own graphs (both key-buffer
    # parities; P2P steps in two halves): warm them up too
    for _ in range(max(2, a.warmup)):
        an.execute_async(da)
    an.wait()
    cached = bool(r.geometry_cached)
    surface_pass = r.surface_pass
    geo = ctx.geometry_info() if cached else None

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    # N > 1: the ranks leave the host barrier up to ~1 ms apart; a device-side
    # barrier (an NCCL all-reduce on the timed stream) right before the start
    # event starts every rank's clock once all GPUs are there, so the max over
    # ranks measures the job, not the host barrier's skew
    dev_group = dist.new_group(backend="nccl") if dist is not None else None
    dev_token = torch.zeros(1, device=f"cuda:{local}")

    def start(ev):
        barrier()
        if dev_group is not None:
            dist.all_reduce(dev_token, group=dev_group)
        ev.record(stream)

    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    stream = torch.cuda.default_stream()
    clocks = ClockSampler(local)
    barrier()
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dev_group is not None:                          # the device barrier's first call (communicator set-up)
        dist.all_reduce(dev_token, group=dev_group)
    # the timed steps use the stream-ordered Execute (nkb_execute_async): no
    # host synchronisation between steps, so host jitter on one rank does not
    # hold up the composite of the others; the last step's report is waited
    # for inside the timed region and must not have overflowed
    start(e0)
    import time as _time
    th0 = _time.perf_counter()
    for _ in range(a.steps):
        an.execute_async(da)
    host_launch_ms = (_time.perf_counter() - th0) * 1e3 / a.steps
    rep_last = an.wait()
    e1.record(stream)
    barrier()
    clk = clocks.stop()
    if rep_last.overflowed:
        raise RuntimeError("a timed step overflowed its triangle buffer (warm-up should have sized it)")
    ms = max_over_ranks(e0.elapsed_time(e1)) / a.steps
    total_points = sum_over_ranks(float(npts))
    value = total_points / (ms / 1e3)
    # the same steps through the synchronous Execute (host sync + report per step)
    start(e0)
    for _ in range(a.steps):
        an.execute(da, fetch_image=False)
    e1.record(stream)
    barrier()
    ms_sync = max_over_ranks(e0.elapsed_time(e1)) / a.steps

    # per-stage breakdown (events around each stage), also the phase CSV
    fused_ms, stages, ntri = [], [], 0
    for _ in range(max(3, min(a.steps, 10))):
        r = an_t.execute(da, fetch_image=False).report
        fused_ms.append(r.ms_fused)
        ntri = r.n_triangles
        stages.append((r.ms_fused, r.ms_raster, r.ms_composite, r.ms_resolve))
    barrier()
    per_rank = [statistics.mean(fused_ms), float(ntri)]
    if dist is not None:
        gathered = [None] * world
        dist.all_gather_object(gathered, per_rank)
        per_rank_fused = [round(g[0], 4) for g in gathered]
        per_rank_tri = [int(g[1]) for g in gathered]
    else:
        per_rank_fused, per_rank_tri = [round(per_rank[0], 4)], [ntri]

    # roofline of the dominant kernel (the surface pass that ran): §8(d)
    # algorithmic bytes -- fields + coordinates + 48 B per emitted triangle --
    # over the event-timed kernel; what the kernel actually moves (a geometry
    # cache included) is reported beside it as traffic_ratio
    peaks, peak_kind = _peaks()
    fused = statistics.mean(fused_ms)
    kernel_name = {1: "stream_kernel", 2: "fused2_kernel"}.get(surface_pass, "fused_kernel")
    alg_bytes = npts * pb["alg"] + 48 * ntri
    achieved = alg_bytes / (fused / 1e3) / 1e9
    if surface_pass == 1:
        kernel_bpp = pb["fields"] + 8 * pb["plane_axes"]
    elif cached:
        kernel_bpp = pb["fields"] + 8 * pb["plane_axes"] + geo["bytes"] / npts
    else:
        kernel_bpp = pb["fields"] + 24
    kernel_bytes = npts * kernel_bpp + 48 * ntri
    prof = _profile_json(f"traffic_{a.config}.json") or {}
    traffic = prof.get("dram_bytes_per_launch")
    fp64 = None
    if world == 1 and pb["need_grad"]:
        probe = _fp64_peak()
        flops = (_profile_json(f"fp64_{a.config}.json") or {}).get(kernel_name)
        fp64 = {"peak_tflops": probe["tflops"] if probe else None, "probe": probe,
                "flops_per_launch": flops}
        if probe and flops:
            fp64["achieved_tflops"] = flops / (fused / 1e3) / 1e12
            fp64["fp64_frac"] = fp64["achieved_tflops"] / probe["tflops"]
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                "kernel": kernel_name, "kernel_ms": fused, "alg_bytes_per_launch": alg_bytes,
                "alg_bytes_per_point": pb["alg"], "triangles": ntri, "peak_source": peak_kind,
                "kernel_bytes_per_point": round(kernel_bpp, 3),
                "traffic_ratio": kernel_bytes / alg_bytes,
                "traffic_source": prof.get("source"),
                "frac_of_nominal_8tbs": achieved / 8000.0}
    if geo is not None:
        roofline["geometry"] = geo
    if fp64 is not None:
        roofline["fp64"] = fp64

    # the same step with the geometry recomputed every step (no cache): reads
    # exactly the algorithmic bytes
    uncached = None
    if cached and world == 1:
        ctx.set_geometry_cache(False)
        for _ in range(2):
            an_t.execute(da, fetch_image=False)
        um = [an_t.execute(da, fetch_image=False).report.ms_fused for _ in range(max(3, min(a.steps, 10)))]
        ctx.set_geometry_cache(True)
        an_t.execute(da, fetch_image=False)
        uk = statistics.mean(um)
        uncached = {"fused_ms": round(uk, 4), "bytes_per_point": pb["alg"],
                    "frac": (npts * pb["alg"] + 48 * ntri) / (uk / 1e3) / 1e9 / peaks["hbm_gbs"]}

    # ---- end-to-end through the reference-facing sink with host buffers ----
    host_bytes = npts * 8 * (3 + sum(comps.values()))
    e2e = None
    if host_bytes <= a.e2e_max_gb * 1e9:
        hc = hcase if hcase is not None else _host_sample(case, case.n_elements)
        names = [("x", hc.x), ("y", hc.y), ("z", hc.z)] + list(hc.fields.items())
        pinned = PinnedBuffer(sum(v.nbytes for _, v in names))
        off, host = 0, {}
        for k, v in names:
            view = np.frombuffer((__import__("ctypes").c_byte * v.nbytes).from_address(pinned.ptr + off),
                                 dtype=np.float64)
            view[:] = v.ravel()
            view.setflags(write=False)          # immutable -> FieldArray aliases the pinned buffer
            host[k] = view.reshape(v.shape)
            off += v.nbytes
        hfields = tuple(FieldArray(k, POINT, hc.fields[k].shape[0], host[k].ravel(), comp_stride=npts)
                        for k in hc.fields)
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
        start(e0)
        for _ in range(e2e_steps):
            sink.consume(Snapshot(0.0, step, rank, (hblk,)))
            step += 1
        sink.flush()
        e1.record(stream)
        barrier()
        e2e_ms = max_over_ranks(e0.elapsed_time(e1)) / e2e_steps
        sink.finalize()
        e2e = {"value": total_points / (e2e_ms / 1e3), "unit": UNIT, "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": int(sink.adaptor.h2d_bytes),
               "d2h_bytes_per_step": int(a.width * a.width * 3 + 15) if rank == 0 else 0,
               "path": "InsituSink.consume(host pinned snapshot) -> H2D -> execute -> D2H PPM -> file"
                       + (" (written synchronously)" if a.e2e_sync_write else
                          " (written on a writer thread, overlapping the next step's H2D; last write waited for)")}
        del pinned
    else:
        e2e = {"value": None, "unit": UNIT, "h2d_bytes_per_step": int(host_bytes), "d2h_bytes_per_step": 0,
               "skipped": f"partition needs {host_bytes / 1e9:.1f} GB of pinned host memory (> --e2e-max-gb)"}

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms, "ms_per_step_sync": ms_sync,
        "higher_is_better": True, "scaling": wl.scaling,
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded NekRS-layout SEM fields, "
                + ("synth.py numpy generator)" if wl.host_generated else "synth_device.py)"),
        "config": config,
        "e2e": e2e,
        "roofline": roofline,
        "fused_uncached": uncached,
        "stages_ms": dict(zip(("fused", "raster", "composite", "resolve"),
                              (round(statistics.mean(x), 4) for x in zip(*stages)))),
        "fused_ms_per_rank": per_rank_fused,
        "triangles_per_rank": per_rank_tri,
        "geometry_cache": ("on: built once per static mesh in "
                           f"{geo_build_ms:.3f} ms during warm-up") if cached else "off/not needed",
        "execute": "stream-ordered nkb_execute_async x K, one nkb_execute_wait (ms_per_step); "
                   "synchronous nkb_execute per step (ms_per_step_sync)",
        "timed_region": ("host barrier, then a device barrier (NCCL all-reduce on the timed stream), then the "
                         "start event on every rank; CUDA events, max over ranks") if world > 1 else
                        "CUDA events on the launch stream, synchronised on both sides",
        # libnekb200 kernels per step on rank 0, counter init included.  1 GPU:
        # counters, K1g|K1|K1s, K2 raster, K3 resolve (+ next key-buffer
        # clear, range words and report in its last CTA).  NCCL composite:
        # counters, K1g, zbuf clear, K2, range words, K3, report (the reduce
        # kernels are NCCL's).  P2P composite: counters, K1g, epoch, wait, zbuf
        # clear, K2, range words, signal, composite, signal, wait, report;
        # stream-ordered P2P steps report in both halves (one more report)
        "gpu_launches": (4 if world == 1 else 7 if os.environ.get("NKB_COMPOSITE") == "nccl" else
                         13 if rep_last.composite_overlapped else 12) * a.steps,
        "composite_overlapped": bool(rep_last.composite_overlapped),
        "host_ms_per_async_launch": host_launch_ms,
        "clocks": clk,
    }
    if a.csv and rank == 0:
        _write_csv(a.csv, a.config, stages, npts, pb["alg"], ntri, peaks["hbm_gbs"])
    if world == 1 and a.config == "c2":
        out["next_rows"] = next_rows(ctx, da, case, hcase, peaks["hbm_gbs"], pipe)
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        out["cpu_baseline"], out["parity"] = cpu_baseline_and_parity(ctx, local, case, hcase, pipe,
                                                                     an.view_for(da), an, da)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if comm is not None:
        comm.close()
    if dist is not None:
        dist.destroy_process_group()


def _write_csv(path, label, stages, npts, alg_bpp, ntri, hbm_gbs):
    """timings.csv in the reference's schema (reporting.py:21-24) and
    phases.csv with gll_points, alg_bytes and roofline_frac per stage."""
    os.makedirs(path, exist_ok=True)
    names = ("fused", "raster", "composite", "resolve")
    with open(os.path.join(path, "timings.csv"), "w", newline="") as f, \
            open(os.path.join(path, "phases.csv"), "w", newline="") as g:
        w, w2 = csv.writer(f), csv.writer(g)
        w.writerow(TIMINGS_HEADER)
        w2.writerow(PHASES_HEADER)
        for step, st in enumerate(stages):
            for name, ms in zip(names, st):
                sec = ms / 1e3
                w.writerow([label, step, name, f"{sec:.9f}"])
                ab = npts * alg_bpp + 48 * ntri if name == "fused" else 0
                frac = ab / sec / 1e9 / hbm_gbs if (ab and sec > 0) else ""
                w2.writerow([label, step, name, f"{sec:.9f}", npts, ab, frac])


def next_rows(ctx, da, case, hcase, hbm_gbs, pipe=None):
    """SURVEY.md §8f rows built after the hot path, measured on the same
    partition: the stats sink (nkb_stats, numpy-exact min/max/mean of every
    field), DSSUM and the GPU checkpoint encoder (legacy-VTK sections)."""
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
    if case.n_elements == 32768:
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
                        "frac_of_hbm": 16 * npts / ms / 1e6 / hbm_gbs,
                        "kernel": "gs_avg_kernel: runs grouped by copy count, one launch",
                        "note": "in-place average of one f64 field: read + write 8 B/pt (algorithmic)"}
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


def _oracle_surfaces(pipe):
    return [("iso", s.field, s.value) if s.kind == "iso" else ("slice", s.normal, s.value) for s in pipe.surfaces]


def cpu_baseline_and_parity(ctx, local, case, hcase, pipe, view, an, da, reps: int = 2):
    """The C oracle port (oracle/sem_oracle.c) times a bounded sample of the
    benchmarked step on all host cores -- the whole partition for C1/C2 --
    and its result is compared bit for bit with the GPU's on the same input
    bytes: image (RGBA), triangle count and colour range."""
    import numpy as np

    from oracle import oracle as orc
    from paper_2312_09888_b200.analysis import InsituAnalysis

    orc.build()
    cores = _cores()
    e_s = min(case.n_elements, 65536)              # bounded sample (~10-30 s of CPU work)
    hs = hcase if (hcase is not None and e_s == case.n_elements) else _host_sample(case, e_s)
    cf = orc.CaseFields(hs.x, hs.y, hs.z, hs.fields)
    surf = _oracle_surfaces(pipe)
    best, res = math.inf, None
    for _ in range(reps):
        t0 = time.perf_counter()
        res = orc.pipeline_mt(cf, surf, pipe.color_field, view, pipe.width, pipe.height, cores)
        best = min(best, time.perf_counter() - t0)
    full = e_s == case.n_elements
    what = "full" if full else f"first {e_s} of {case.n_elements} elements of the"
    base = {"value": e_s * NN / best, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{what} step (adaptor+Q+iso/slice+raster+resolve), best of {reps}, C oracle port, "
                      f"{cores} threads", "ms_per_step": best * 1e3, "inputs_digest": _case_digest(hs)}
    # the GPU on the same elements, same camera
    from dataclasses import replace

    if full:
        g = an.execute(da, fetch_image=True)
    else:
        from paper_2312_09888_b200.context import Context

        sub = Context(local)
        sda = _sem_adaptor(sub, case, 0, n_elements=e_s)
        g = InsituAnalysis(replace(pipe, view=tuple(view))).execute(sda, fetch_image=True)
    rgba, ntri, rng = res[0], res[2], res[3]
    par = {
        "sample": "benchmarked partition" if full else f"first {e_s} elements",
        "image": bool(np.array_equal(g.rgba, rgba)),
        "ntri": bool(g.report.n_triangles == ntri),
        "range": bool(np.array_equal(np.array(g.report.range).view(np.uint64), np.array(rng).view(np.uint64))),
        "triangles": int(ntri),
        "differing_pixels": int(np.count_nonzero(np.any(g.rgba != rgba, axis=-1))),
        "oracle": "oracle/sem_oracle.c orc_pipeline_mt",
    }
    par["ok"] = par["image"] and par["ntri"] and par["range"]
    return base, par


# ---------------------------------------------------------------------------
# reference arm: the CPU oracle port on the same workload and bytes
# ---------------------------------------------------------------------------

def run_reference(a):
    rank, world, _ = _env_rank()
    if rank != 0:
        return
    from oracle import oracle as orc
    from paper_2312_09888_b200 import synth
    from paper_2312_09888_b200.analysis import ortho_view

    orc.build()
    cores = _cores()
    wl = Workload(a, world)
    pipe = _pipeline(wl.params, a.width)
    # bounded sample: ~2 s worth of elements per step (measured ~1.3M pts/s per
    # thread), taken from the start of rank 0's partition -- for c1/c2 at one
    # GPU the whole partition, i.e. the very bytes our arm renders
    e_rank0 = synth.partition(wl.n_global, 0, world)[1]
    e_sample = min(e_rank0, max(64, int(2.0 * 1.3e6 * cores / NN)))
    case = synth.CONFIGS[a.config](0, e_sample, wl.scale)
    cf = orc.CaseFields(case.x, case.y, case.z, case.fields)
    if e_sample == e_rank0 and world == 1:
        b = (case.x.min(), case.x.max(), case.y.min(), case.y.max(), case.z.min(), case.z.max())
    else:
        b = synth_bounds(a.config, wl.scale)
    view = ortho_view(b, pipe.width, pipe.height, *pipe.view_dir)
    surf = _oracle_surfaces(pipe)
    for _ in range(a.warmup):
        orc.pipeline_mt(cf, surf, pipe.color_field, view, pipe.width, pipe.height, cores)
    t0 = time.perf_counter()
    for _ in range(a.steps):
        orc.pipeline_mt(cf, surf, pipe.color_field, view, pipe.width, pipe.height, cores)
    dt = (time.perf_counter() - t0) / a.steps
    v = e_sample * NN / dt
    sample = (f"{e_sample} of {wl.n_global} elements of {a.config} per step (start of rank 0's partition), "
              f"full pipeline, C oracle port on {cores} threads")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": wl.scaling,
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded NekRS-layout SEM fields, synth.py numpy generator)",
        "config": common_config(wl, a),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
                         "inputs_digest": _case_digest(case)},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def synth_bounds(config, scale):
    """Bounding box of a whole config (for the reference arm's camera when it
    renders only a sample)."""
    from paper_2312_09888_b200 import synth

    if config == "c1":
        return (0.0, 2 * math.pi) * 3
    if config == "c2":
        return (-1.0, 1.0, -1.0, 1.0, 0.0, 1.0)
    if config == "c3":
        return (-1.0, 1.0, -1.0, 1.0, 0.0, 20.0 * scale)
    if config == "c4":
        return (0.0, 1.0) * 3
    nel = synth.c5_lattice(scale)
    h = math.pi / 8.0
    return (0.0, h * nel[0], 0.0, h * nel[1], 0.0, h * nel[2])


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="c2/c3: weak (one config per GPU) or strong (one config split over the GPUs)")
    ap.add_argument("--elements", type=int, default=0, help="c5: elements of the box (default 65536 x N)")
    ap.add_argument("--width", type=int, default=1024)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--csv", default="", help="directory for timings.csv / phases.csv")
    ap.add_argument("--e2e-max-gb", type=float, default=12.0)
    ap.add_argument("--partition", default="equal", choices=["equal", "work"],
                    help="N>1 device-generated configs: equal contiguous element ranges (the solver's "
                         "partition) or ranges balancing the surface-pass cost")
    ap.add_argument("--e2e-sync-write", action="store_true", help="write each PPM inside consume() (no writer thread)")
    a = ap.parse_args()
    if a.warmup < 3:
        a.warmup = 3
    if a.config == "c2" and a.scaling == "strong":
        ap.error("c2 is weak-scaled only (configs[1] per GPU)")
    ws = os.environ.get("WORLD_SIZE")
    if ws is not None and int(ws) != a.gpus:
        print(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={ws}", file=sys.stderr)
        sys.exit(2)
    if ws is None and a.gpus > 1:
        # spawn one rank per GPU ourselves (torchrun, loopback rendezvous)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
               os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.run(cmd).returncode)
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
