"""Kernel-level A/B timing of the in situ step (device-generated inputs, no
e2e / oracle legs): median per-stage CUDA-event times over --reps steps.

    NKB_LIB=path/to/libnekb200.so python tools/kbench.py c2 c3 --reps 30
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--elements", type=int, default=65536, help="c5 box size")
    ap.add_argument("--width", type=int, default=1024)
    ap.add_argument("--geo", default="auto", choices=["auto", "full", "off"])
    ap.add_argument("--tag", default=os.path.basename(os.environ.get("NKB_LIB", "libnekb200.so")))
    a = ap.parse_args()
    import torch

    from paper_2312_09888_b200 import synth_device
    from paper_2312_09888_b200.adaptor import SemDataAdaptor
    from paper_2312_09888_b200.analysis import InsituAnalysis, pipeline_from_params
    from paper_2312_09888_b200.context import Context
    from paper_2312_09888_b200.data_model import POINT, FieldArray, SemBlock, Snapshot
    from dataclasses import replace

    ctx = Context(0)
    ctx.set_geometry_cache({"auto": "auto", "full": "full", "off": False}[a.geo])
    for cfg in a.configs:
        scale = a.elements if cfg == "c5" else 1
        case = synth_device.make_case(cfg, 0, 1, scale=scale, device="cuda:0")
        if case is None:                  # c1: the numpy generator's case, copied to the device
            from types import SimpleNamespace

            from paper_2312_09888_b200 import synth

            h = synth.make_case(cfg, 0, 1)
            dev = lambda a_: torch.from_numpy(a_).to("cuda:0")
            case = SimpleNamespace(n_elements=h.n_elements, n_points=h.n_points, x=dev(h.x), y=dev(h.y), z=dev(h.z),
                                   fields={k: dev(v) for k, v in h.fields.items()}, params=h.params)
        torch.cuda.synchronize()
        fields = tuple(FieldArray(k, POINT, v.shape[0], v.reshape(-1), comp_stride=case.n_points)
                       for k, v in case.fields.items())
        da = SemDataAdaptor(ctx)
        da.initialize(Snapshot(0.0, 0, 0, (SemBlock(case.n_elements, case.x, case.y, case.z, fields=fields),)))
        pipe = replace(pipeline_from_params({**case.params, "width": str(a.width), "height": str(a.width)}),
                       timing=True)
        an = InsituAnalysis(pipe)
        for _ in range(3):
            an.execute(da, fetch_image=False)
        reps = [an.execute(da, fetch_image=False).report for _ in range(a.reps)]
        med = lambda k: round(statistics.median(getattr(r, k) for r in reps), 4)
        print(json.dumps({"tag": a.tag, "config": cfg, "E": case.n_elements, "pass": reps[-1].surface_pass,
                          "geo": ctx.geometry_info()["layout"], "fused": med("ms_fused"), "raster": med("ms_raster"),
                          "resolve": med("ms_resolve"), "ntri": reps[-1].n_triangles}), flush=True)
        del da, case
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
