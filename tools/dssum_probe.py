"""DSSUM timing probe on the C2 lattice (32^3 elements, 16.8M GLL copies):
one-pass vs two-pass kernels, CUDA-event timed; under ncu it launches each
variant a few times (``-k regex:gs_``)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_09888_b200 import synth, synth_device  # noqa: E402
from paper_2312_09888_b200.adaptor import SemDataAdaptor  # noqa: E402
from paper_2312_09888_b200.context import Context  # noqa: E402
from paper_2312_09888_b200.data_model import POINT, FieldArray, SemBlock, Snapshot  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    case = synth_device.make_case("c2", 0, 1, device="cuda:0")
    ctx = Context(0)
    da = SemDataAdaptor(ctx)
    fields = tuple(FieldArray(k, POINT, v.shape[0], v.reshape(-1), comp_stride=case.n_points)
                   for k, v in case.fields.items())
    da.initialize(Snapshot(0.0, 0, 0, (SemBlock(case.n_elements, case.x, case.y, case.z, fields=fields),)))
    gid = torch.from_numpy(synth.lattice_ids((32, 32, 32), 0, 32768)).cuda()
    ctx.mesh_set_global_ids(gid)
    f = case.fields["temperature"].reshape(-1).clone()
    out = {}
    for name, env in (("one_pass", None), ("two_pass", "1")):
        if env:
            os.environ["NKB_DSSUM_TWO_PASS"] = env
        else:
            os.environ.pop("NKB_DSSUM_TWO_PASS", None)
        ctx.dssum(f)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            ctx.dssum(f)
        e1.record()
        torch.cuda.synchronize()
        out[name] = e0.elapsed_time(e1) / reps
    out["points"] = case.n_points
    print(json.dumps(out))
    ctx.close()


if __name__ == "__main__":
    main()
