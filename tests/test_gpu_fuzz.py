"""Randomised parity (hypothesis): random element lattices, fields, surfaces,
colour fields, cameras and image sizes -- GPU triangles (ordered mode),
images and depth bit-identical to the oracle.  Includes iso values placed
exactly on node values (the `>=` inside rule) and degenerate fields."""
import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from oracle import oracle as O
from paper_2312_09888_b200 import synth
from paper_2312_09888_b200.adaptor import SemDataAdaptor
from paper_2312_09888_b200.analysis import InsituAnalysis, Pipeline, Surface
from paper_2312_09888_b200.data_model import POINT, FieldArray, SemBlock, Snapshot

pytestmark = pytest.mark.gpu

_CTX = {}


def _ctx():
    if "c" not in _CTX:
        from paper_2312_09888_b200.context import Context

        _CTX["c"] = Context(0)
    return _CTX["c"]


@st.composite
def scenarios(draw):
    nel = (draw(st.integers(1, 3)), draw(st.integers(1, 3)), draw(st.integers(1, 2)))
    seed = draw(st.integers(0, 10_000))
    kinds = draw(st.lists(st.sampled_from(["Q", "temperature", "vorticity:mag", "velocity:mag", "slice", "snap"]),
                          min_size=0, max_size=4))
    color = draw(st.sampled_from(["temperature", "Q", "vorticity:mag", "velocity:mag"]))
    w, h = draw(st.integers(1, 96)), draw(st.integers(1, 96))
    az, el = draw(st.floats(-180, 180)), draw(st.floats(-80, 80))
    proj = draw(st.sampled_from(["ortho", "perspective"]))
    fov = draw(st.floats(5.0, 120.0))
    return nel, seed, kinds, color, w, h, az, el, proj, fov


@settings(max_examples=150, deadline=None, suppress_health_check=list(HealthCheck))
@given(scenarios())
def test_random_pipelines_bit_exact(sc):
    nel, seed, kinds, color, w, h, az, el, proj, fov = sc
    case = synth.box(nel=nel, seed=seed)
    rng = np.random.default_rng(seed)
    surfaces, orc = [], []
    for k in kinds:
        if k == "slice":
            n = tuple(float(v) for v in rng.uniform(-1, 1, 3))
            if n == (0.0, 0.0, 0.0):
                n = (0.0, 0.0, 1.0)
            d = float(rng.uniform(-0.5, 1.5))
            surfaces.append(Surface("slice", value=d, normal=n))
            orc.append(("slice", n, d))
        elif k == "snap":                           # iso exactly on a node value of temperature
            v = float(case.fields["temperature"][0, rng.integers(case.n_points)])
            surfaces.append(Surface("iso", "temperature", v))
            orc.append(("iso", "temperature", v))
        else:
            v = float(rng.uniform(-1.0, 1.5))
            surfaces.append(Surface("iso", k, v))
            orc.append(("iso", k, v))
    ctx = _ctx()
    da = SemDataAdaptor(ctx)
    fields = tuple(FieldArray(k, POINT, v.shape[0], v.ravel(), comp_stride=case.n_points)
                   for k, v in case.fields.items())
    da.initialize(Snapshot(0.0, 0, 0, (SemBlock(case.n_elements, case.x, case.y, case.z, fields=fields),)))
    pipe = Pipeline(surfaces=tuple(surfaces), color_field=color, width=w, height=h, view_dir=(az, el),
                    emit_meta=True, projection=proj, fov=fov)
    res = InsituAnalysis(pipe).execute(da, depth=True)
    cf = O.CaseFields(case.x, case.y, case.z, case.fields)
    tri, meta, (cmin, cmax) = O.mc(cf, orc, color)
    gt, gm = ctx.triangles(with_meta=True)
    assert res.report.n_triangles == len(tri)
    assert np.array_equal(gm, meta)
    assert np.array_equal(gt.view(np.uint32), tri.view(np.uint32))
    assert res.report.range == (cmin, cmax)
    z = O.raster(tri, res.view, w, h)
    rgba, dep = O.resolve(z, w, h, cmin, cmax)
    assert np.array_equal(res.rgba, rgba)
    assert np.array_equal(res.depth.view(np.uint32), dep.view(np.uint32))


def test_nan_field_values_match_oracle():
    """NaN nodes: outside every iso (NaN >= v is false), ignored by the colour
    range (fmin/fmax), NaN colour scalars resolve to channel 0 -- GPU and
    oracle agree bit for bit."""
    case = synth.box(nel=(2, 2, 1), seed=3)
    t = case.fields["temperature"]
    t[0, ::97] = np.nan
    ctx = _ctx()
    da = SemDataAdaptor(ctx)
    fields = tuple(FieldArray(k, POINT, v.shape[0], v.ravel(), comp_stride=case.n_points)
                   for k, v in case.fields.items())
    da.initialize(Snapshot(0.0, 0, 0, (SemBlock(case.n_elements, case.x, case.y, case.z, fields=fields),)))
    pipe = Pipeline(surfaces=(Surface("iso", "temperature", 0.6), Surface("iso", "Q", 0.5)),
                    color_field="temperature", width=64, height=48, emit_meta=True)
    res = InsituAnalysis(pipe).execute(da, depth=True)
    cf = O.CaseFields(case.x, case.y, case.z, case.fields)
    tri, meta, (cmin, cmax) = O.mc(cf, [("iso", "temperature", 0.6), ("iso", "Q", 0.5)], "temperature")
    gt, gm = ctx.triangles(with_meta=True)
    assert np.array_equal(gm, meta) and np.array_equal(gt.view(np.uint32), tri.view(np.uint32))
    assert res.report.range == (cmin, cmax)
    z = O.raster(tri, res.view, 64, 48)
    rgba, dep = O.resolve(z, 64, 48, cmin, cmax)
    assert np.array_equal(res.rgba, rgba) and np.array_equal(res.depth.view(np.uint32), dep.view(np.uint32))
