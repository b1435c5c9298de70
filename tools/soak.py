"""Soak: many bridge steps (insitu + stats + checkpoint sinks) on one mesh;
device memory must stay flat (no per-step allocations leak)."""
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2312_09888_b200 import synth  # noqa: E402
from paper_2312_09888_b200.bridge import initialize, parse_config  # noqa: E402
from paper_2312_09888_b200.data_model import POINT, FieldArray, SemBlock, Snapshot  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 300
case = synth.rbc_cylinder(nel=(8, 8, 8))
d = tempfile.mkdtemp()
doc = (f'<sensei><analysis type="insitu" frequency="1" dir="{d}/img" iso="temperature=0.5;Q=1.0" slice="y=0" '
       f'field="temperature" width="256" height="256" view="-60,25"/>'
       f'<analysis type="stats" frequency="1" path="{d}/s.csv"/>'
       f'<analysis type="checkpoint" frequency="50" dir="{d}/ck" arrays="Q"/></sensei>')
br = initialize(parse_config(doc))
rng = np.random.default_rng(0)
fields = lambda: tuple(FieldArray(k, POINT, v.shape[0], (v + 0.01 * rng.standard_normal(v.shape)).ravel(),  # noqa: E731
                                  comp_stride=case.n_points) for k, v in case.fields.items())
x, y, z = (np.array(a) for a in (case.x, case.y, case.z))
for a in (x, y, z):
    a.flags.writeable = False
free0 = None
for st in range(steps):
    blk = SemBlock(case.n_elements, x, y, z, fields=fields())
    reps = br.update(Snapshot(0.01 * st, st, 0, (blk,)))
    assert all(r.error is None for r in reps), reps
    if st == 20:
        torch.cuda.synchronize()
        free0 = torch.cuda.mem_get_info()[0]
torch.cuda.synchronize()
free1 = torch.cuda.mem_get_info()[0]
print(f"steps={steps} device free delta after warm-up: {(free0 - free1) / 1e6:.1f} MB")
assert abs(free0 - free1) < 64e6, "device memory grows with steps"
print("soak ok")
