"""Small workload that launches every hot-path kernel once, for
compute-sanitizer (memcheck / racecheck / synccheck, one tool per run):

  K0 geometry (compact + full), K1g (fast + ordered, node program and generic),
  K1 (uncached), K1s (no gradient), K2 raster, K3 resolve, range/report
  kernels, the P2P composite kernel over in-process partitions, the stats and
  DSSUM kernels, GetMesh / AddArray exports.

    compute-sanitizer --tool memcheck python tools/sanitize_case.py
"""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402


def main():
    import torch

    from paper_2312_09888_b200 import synth
    from paper_2312_09888_b200.adaptor import SemDataAdaptor
    from paper_2312_09888_b200.analysis import InsituAnalysis, Pipeline, Surface, ortho_view
    from paper_2312_09888_b200.context import Context
    from paper_2312_09888_b200.data_model import POINT, FieldArray, SemBlock, Snapshot

    case = synth.rbc_cylinder(nel=(3, 3, 4))           # 36 curved, extruded elements
    b = (case.x.min(), case.x.max(), case.y.min(), case.y.max(), case.z.min(), case.z.max())
    view = ortho_view(b, 96, 80, -60.0, 25.0)

    def block(c, e0, e1):
        n0, n1 = e0 * 512, e1 * 512
        f = tuple(FieldArray(k, POINT, v.shape[0], np.ascontiguousarray(v[:, n0:n1]).ravel(), comp_stride=n1 - n0)
                  for k, v in c.fields.items())
        return SemBlock(e1 - e0, c.x[n0:n1], c.y[n0:n1], c.z[n0:n1], fields=f, element_offset=e0,
                        n_elements_global=c.n_elements)

    pipes = [
        Pipeline(surfaces=(Surface("iso", "temperature", 0.5), Surface("iso", "Q", 1.0),
                           Surface("slice", value=0.0, normal=(0, 1, 0))), color_field="temperature",
                 width=96, height=80, view=view, composite=False),                        # K1g node program
        Pipeline(surfaces=(Surface("iso", "vorticity:mag", 1.0),), color_field="Q", width=96, height=80,
                 view=view, composite=False, emit_meta=True),                             # K1g generic, ordered
        Pipeline(surfaces=(Surface("iso", "velocity:mag", 0.4), Surface("slice", value=0.5, normal=(0, 0, 1))),
                 color_field="velocity:mag", width=96, height=80, view=view, composite=False),   # K1s
    ]
    ctx = Context(0)
    da = SemDataAdaptor(ctx)
    da.initialize(Snapshot(0.0, 0, 0, (block(case, 0, case.n_elements),)))
    for mode in ("auto", "full", False):
        ctx.set_geometry_cache(mode)
        for p in pipes:
            r = InsituAnalysis(p).execute(da, depth=True)
            print(mode, p.color_field, r.report.surface_pass, r.report.n_triangles, flush=True)
    ctx.set_geometry_cache(True)
    # exports (AddArray / GetMesh), stats, DSSUM
    q = torch.empty(case.n_points, dtype=torch.float64, device="cuda")
    ctx.add_array("Q", q)
    g = da.get_mesh()
    print("mesh", g.n_points if hasattr(g, "n_points") else "ok")
    print("stats", ctx.stats([da.field_segment("velocity")]))
    gid = torch.from_numpy(synth.lattice_ids((3, 3, 4), 0, case.n_elements)).cuda()
    ctx.mesh_set_global_ids(gid)
    t = torch.from_numpy(np.ascontiguousarray(case.fields["temperature"][0])).cuda()
    ctx.dssum(t)
    # in-process partition composite (the P2P composite kernel)
    parts = []
    for r in range(3):
        e0, e1 = synth.partition(case.n_elements, r, 3)
        c = Context(0)
        d = SemDataAdaptor(c)
        d.initialize(Snapshot(0.0, 0, r, (block(case, e0, e1),)))
        InsituAnalysis(pipes[0]).execute(d, fetch_image=False)
        parts.append((c, d))
    parts[0][0].composite_partitions([c for c, _ in parts], pipes[0].native(view))
    print("composite", parts[0][0].image(96, 80).sum())
    torch.cuda.synchronize()
    print("sanitize case done")


if __name__ == "__main__":
    main()
