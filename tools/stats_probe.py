"""Time nkb_stats (numpy-exact min/max/mean) on device-resident SEM fields.

    python tools/stats_probe.py [c2|c4] [--reps 10]

Prints per-field wall time per call (plan cached) and the aggregate GB/s.
"""
from __future__ import annotations

import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2312_09888_b200 import synth_device  # noqa: E402
from paper_2312_09888_b200.adaptor import SemDataAdaptor  # noqa: E402
from paper_2312_09888_b200.context import Context  # noqa: E402
from paper_2312_09888_b200.data_model import POINT, FieldArray, SemBlock, Snapshot  # noqa: E402


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
    tot_b, tot_t = 0, 0.0
    for n in case.fields:
        seg = [da.field_segment(n)]
        r = ctx.stats(seg)
        t0 = time.perf_counter()
        for _ in range(a.reps):
            r = ctx.stats(seg)
        dt = (time.perf_counter() - t0) / a.reps
        nb = 8 * case.fields[n].shape[0] * case.n_points
        tot_b += nb
        tot_t += dt
        print(f"{a.config} {n}: {nb / 1e6:.0f} MB {dt * 1e3:.3f} ms {nb / dt / 1e9:.0f} GB/s -> {r}", flush=True)
    print(f"{a.config} all fields: {tot_b / 1e6:.0f} MB {tot_t * 1e3:.3f} ms {tot_b / tot_t / 1e9:.0f} GB/s")


if __name__ == "__main__":
    main()
