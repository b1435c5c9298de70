"""Time the GetMesh / AddArray export kernels (R11 explicit VTK form) on a
device-resident config, in GB/s of algorithmic bytes.

    python tools/export_probe.py [c2] [--reps 10]
"""
from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2312_09888_b200 import synth_device  # noqa: E402
from paper_2312_09888_b200.adaptor import SemDataAdaptor  # noqa: E402
from paper_2312_09888_b200.context import Context  # noqa: E402
from paper_2312_09888_b200.data_model import POINT, FieldArray, SemBlock, Snapshot  # noqa: E402
from paper_2312_09888_b200.device import DeviceArray  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="c2")
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    case = synth_device.make_case(a.config, 0, 1, device="cuda:0")
    ctx = Context(0)
    da = SemDataAdaptor(ctx)
    fields = tuple(FieldArray(k, POINT, v.shape[0], v.reshape(-1), comp_stride=case.n_points)
                   for k, v in case.fields.items())
    da.initialize(Snapshot(0.0, 0, 0, (SemBlock(case.n_elements, case.x, case.y, case.z, fields=fields),)))
    m = ctx.metadata()
    npts, ncells = int(m.n_points), int(m.n_cells)
    pts = DeviceArray.empty(ctx, (npts, 3), np.float64)
    conn = DeviceArray.empty(ctx, (ncells, 8), np.int64)
    offs = DeviceArray.empty(ctx, (ncells + 1,), np.int64)
    types = DeviceArray.empty(ctx, (ncells,), np.uint8)
    vel = DeviceArray.empty(ctx, (3 * npts,), np.float64)

    def timed(fn, nbytes, label):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        print(f"{a.config} {label}: {nbytes / 1e9:.2f} GB {ms:.3f} ms {nbytes / ms / 1e6:.0f} GB/s", flush=True)

    timed(lambda: ctx.get_mesh(pts, None, None, None), 48 * npts, "GetMesh points (24 B read + 24 B written /pt)")
    timed(lambda: ctx.get_mesh(None, conn, offs, types), 73 * ncells, "GetMesh connectivity+offsets+types (73 B/cell)")
    timed(lambda: ctx.add_array("velocity", vel), 48 * npts, "AddArray velocity AoS (24 B read + 24 B written /pt)")


if __name__ == "__main__":
    main()
