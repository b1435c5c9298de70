"""Break the bench's e2e step (InsituSink.consume with pinned host buffers)
into its parts, C2 by default.

    python tools/e2e_probe.py [c2] [--steps 5]
"""
from __future__ import annotations

import argparse
import ctypes
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2312_09888_b200 import synth_device  # noqa: E402
from paper_2312_09888_b200.data_model import POINT, FieldArray, SemBlock, Snapshot  # noqa: E402
from paper_2312_09888_b200.device import PinnedBuffer  # noqa: E402
from paper_2312_09888_b200.sinks import ImageRGB, InsituSink, write_ppm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="c2")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--width", type=int, default=1024)
    a = ap.parse_args()
    case = synth_device.make_case(a.config, 0, 1, device="cuda:0").to_host()
    npts = case.n_points
    names = [("x", case.x), ("y", case.y), ("z", case.z)] + list(case.fields.items())
    pinned = PinnedBuffer(sum(v.nbytes for _, v in names))
    off, host = 0, {}
    for k, v in names:
        view = np.frombuffer((ctypes.c_byte * v.nbytes).from_address(pinned.ptr + off), dtype=np.float64)
        view[:] = v.ravel()
        view.setflags(write=False)
        host[k] = view.reshape(v.shape)
        off += v.nbytes
    fields = tuple(FieldArray(k, POINT, case.fields[k].shape[0], host[k].ravel(), comp_stride=npts)
                   for k in case.fields)
    blk = SemBlock(case.n_elements, host["x"], host["y"], host["z"], fields=fields)
    field_bytes = sum(v.nbytes for k, v in case.fields.items())

    # raw pinned H2D bandwidth of the same bytes (torch, one copy)
    src = torch.from_numpy(np.frombuffer((ctypes.c_byte * field_bytes).from_address(pinned.ptr + 3 * 8 * npts),
                                         dtype=np.uint8))
    dst = torch.empty(field_bytes, dtype=torch.uint8, device="cuda")
    for _ in range(2):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    bw = 3 * field_bytes / (time.perf_counter() - t0) / 1e9
    print(f"raw pinned H2D: {field_bytes / 1e6:.0f} MB at {bw:.1f} GB/s -> {field_bytes / bw / 1e6:.2f} ms")

    d = tempfile.mkdtemp()
    params = {**case.params, "width": str(a.width), "height": str(a.width), "dir": d}
    sink = InsituSink(params)
    for st in range(2):
        sink.consume(Snapshot(0.0, st, 0, (blk,)))
    T = {"initialize(H2D)": 0.0, "execute": 0.0, "image D2H": 0.0, "rgb bytes": 0.0, "write_ppm": 0.0}
    t_all = time.perf_counter()
    for st in range(2, 2 + a.steps):
        s = Snapshot(0.0, st, 0, (blk,))
        t = time.perf_counter()
        sink.adaptor.initialize(s)
        torch.cuda.synchronize()
        T["initialize(H2D)"] += time.perf_counter() - t
        t = time.perf_counter()
        res = sink.analysis.execute(sink.adaptor, fetch_image=False)
        torch.cuda.synchronize()
        T["execute"] += time.perf_counter() - t
        t = time.perf_counter()
        rgba = sink.adaptor.ctx.image(sink.pipeline.width, sink.pipeline.height)
        T["image D2H"] += time.perf_counter() - t
        t = time.perf_counter()
        b = rgba[..., :3].tobytes()
        T["rgb bytes"] += time.perf_counter() - t
        t = time.perf_counter()
        write_ppm(ImageRGB(sink.pipeline.width, sink.pipeline.height, b), os.path.join(d, f"s{st}.ppm"))
        T["write_ppm"] += time.perf_counter() - t
    tot = (time.perf_counter() - t_all) / a.steps * 1e3
    print(f"h2d bytes/step {sink.adaptor.h2d_bytes}; total {tot:.2f} ms/step")
    for k, v in T.items():
        print(f"  {k:18s} {v / a.steps * 1e3:8.3f} ms")
    t = time.perf_counter()
    for st in range(a.steps):
        sink.consume(Snapshot(0.0, 100 + st, 0, (blk,)))
    print(f"sink.consume: {(time.perf_counter() - t) / a.steps * 1e3:.2f} ms/step")


if __name__ == "__main__":
    main()
