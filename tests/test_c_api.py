"""The ABI from plain C (examples/insitu_c_api.c, built by build()): the
image a C caller gets equals the Python path's and the oracle's, byte for
byte, on the same inputs."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2312_09888_b200", "lib", "insitu_c_api")


def test_example_is_built():
    assert os.path.exists(BIN), "build() links examples/insitu_c_api.c against libnekb200"


@pytest.mark.gpu
def test_c_caller_image_equals_python_and_oracle(tmp_path):
    from oracle import oracle as O
    from paper_2312_09888_b200.adaptor import SemDataAdaptor
    from paper_2312_09888_b200.analysis import InsituAnalysis, Pipeline, Surface
    from paper_2312_09888_b200.context import Context
    from paper_2312_09888_b200.data_model import POINT, FieldArray, SemBlock, Snapshot

    r = subprocess.run([BIN, str(tmp_path / "c.ppm"), str(tmp_path / "f.bin")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    c_ppm = (tmp_path / "c.ppm").read_bytes()
    h = np.fromfile(tmp_path / "f.bin", dtype=np.float64).reshape(7, -1)
    x, y, z, vel, t = h[0], h[1], h[2], h[3:6], h[6]
    E = x.size // 512
    ctx = Context(0)
    da = SemDataAdaptor(ctx)
    fields = (FieldArray("velocity", POINT, 3, vel.ravel(), comp_stride=x.size), FieldArray("temperature", POINT, 1, t))
    da.initialize(Snapshot(0.0, 0, 0, (SemBlock(E, x, y, z, fields=fields),)))
    view = (70.0, 0.0, 0.0, 10.0, 0.0, -70.0, 0.0, 110.0, 0.0, 0.0, -0.5, 1.0)
    surf = (Surface("iso", "Q", 0.5), Surface("iso", "temperature", 0.6),
            Surface("slice", value=0.75, normal=(0.0, 1.0, 0.0)))
    res = InsituAnalysis(Pipeline(surfaces=surf, color_field="temperature", width=160, height=120,
                                  view=view)).execute(da)
    assert bytes(ctx.image_ppm()) == c_ppm
    cf = O.CaseFields(x, y, z, {"velocity": vel, "temperature": t[None]})
    rgba, _, ntri, rng = O.pipeline_mt(cf, [("iso", "Q", 0.5), ("iso", "temperature", 0.6),
                                            ("slice", (0.0, 1.0, 0.0), 0.75)], "temperature", view, 160, 120, 2)
    assert res.report.n_triangles == ntri and c_ppm[len(b"P6\n160 120\n255\n"):] == rgba[..., :3].tobytes()
    ctx.close()
