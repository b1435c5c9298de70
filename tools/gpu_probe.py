"""Ad-hoc GPU probe: parity of a config against the oracle + per-stage timing.

    python tools/gpu_probe.py c2 [--oracle] [--reps 5]
"""
from __future__ import annotations

import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2312_09888_b200 import synth  # noqa: E402
from paper_2312_09888_b200.adaptor import SemDataAdaptor  # noqa: E402
from paper_2312_09888_b200.analysis import InsituAnalysis, pipeline_from_params  # noqa: E402
from paper_2312_09888_b200.context import Context  # noqa: E402
from paper_2312_09888_b200.data_model import POINT, FieldArray, SemBlock, Snapshot  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", default="c2", nargs="?")
    ap.add_argument("--oracle", action="store_true")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--width", type=int, default=1024)
    ap.add_argument("--no-surfaces", action="store_true")
    ap.add_argument("--color", default=None)
    ap.add_argument("--geo", choices=("on", "off", "both"), default="both")
    ap.add_argument("--device-gen", action="store_true", help="generate the case on the GPU (fast; no --oracle)")
    a = ap.parse_args()
    t0 = time.time()
    if a.device_gen:
        from paper_2312_09888_b200 import synth_device
        case = synth_device.make_case(a.config, 0, 1, device="cuda:0")
    else:
        case = synth.make_case(a.config) if a.config != "box" else synth.box()
    print(f"[{a.config}] E={case.n_elements} pts={case.n_points} gen {time.time()-t0:.1f}s", flush=True)
    ctx = Context(0)
    da = SemDataAdaptor(ctx)
    fields = tuple(FieldArray(k, POINT, v.shape[0], v.reshape(-1), comp_stride=case.n_points)
                   for k, v in case.fields.items())
    blk = SemBlock(case.n_elements, case.x, case.y, case.z, fields=fields)
    da.initialize(Snapshot(0.0, 0, 0, (blk,)))
    params = dict(case.params)
    params["width"] = params["height"] = str(a.width)
    pipe = pipeline_from_params(params)
    from dataclasses import replace
    pipe = replace(pipe, timing=True, emit_meta=a.oracle)
    if a.no_surfaces:
        pipe = replace(pipe, surfaces=())
    if a.color:
        pipe = replace(pipe, color_field=a.color)
    an = InsituAnalysis(pipe)
    plane = any(s.kind == "slice" for s in pipe.surfaces)
    images = {}
    for geo in (("on", "off") if a.geo == "both" else (a.geo,)):
        ctx.set_geometry_cache(geo == "on")
        for r in range(a.reps):
            res = an.execute(da)
            rp = res.report
            tot = rp.ms_fused + rp.ms_raster + rp.ms_composite + rp.ms_resolve
            bpp = 8 * sum(v.shape[0] for v in case.fields.values())
            bpp += (24 if (not rp.geometry_cached or plane) else 0) + (72 if rp.geometry_cached else 0)
            gb = case.n_points * bpp / 1e9
            print(f"geo={geo} rep {r}: ntri={rp.n_triangles} fused {rp.ms_fused:.3f} ms ({gb / rp.ms_fused * 1e3:.0f} GB/s"
                  f" of {gb:.2f} GB) raster {rp.ms_raster:.3f} resolve {rp.ms_resolve:.3f} total {tot:.3f} ms "
                  f"range {rp.range} reran={rp.reran} cached={rp.geometry_cached} build={rp.ms_geometry:.3f}",
                  flush=True)
        images[geo] = res.rgba.copy()
    if len(images) == 2:
        print("cached == uncached image:", np.array_equal(images["on"], images["off"]))
    if a.oracle:
        from oracle import oracle as orc
        cf = orc.CaseFields(case.x, case.y, case.z, case.fields)
        surfaces = []
        for s in pipe.surfaces:
            surfaces.append(("iso", s.field, s.value) if s.kind == "iso" else ("slice", s.normal, s.value))
        t0 = time.time()
        rgba, dep, ntri, rng = orc.pipeline_mt(cf, surfaces, pipe.color_field, res.view, pipe.width,
                                               pipe.height, os.cpu_count() or 8)
        print(f"oracle {time.time()-t0:.1f}s on {os.cpu_count()} threads: ntri={ntri} range={rng}")
        print("ntri equal:", ntri == rp.n_triangles, " image equal:", np.array_equal(rgba, res.rgba),
              " mismatched px:", int(np.sum(np.any(rgba != res.rgba, axis=-1))))
        os.makedirs("gpurun_out", exist_ok=True)
        np.save(f"gpurun_out/{a.config}_gpu.npy", res.rgba)
        np.save(f"gpurun_out/{a.config}_orc.npy", rgba)


if __name__ == "__main__":
    main()
