"""DSSUM on one GPU against the oracle, and the
continuous pipeline (Q averaged across element faces before the isosurface)
against the oracle's marching cubes on the averaged field."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2312_09888_b200 import synth
from paper_2312_09888_b200.adaptor import SemDataAdaptor
from paper_2312_09888_b200.analysis import InsituAnalysis, Pipeline, Surface
from paper_2312_09888_b200.data_model import POINT, FieldArray, SemBlock, Snapshot
from paper_2312_09888_b200.device import DeviceArray

pytestmark = pytest.mark.gpu


def _snapshot(case, gid=True):
    fields = tuple(FieldArray(k, POINT, v.shape[0], v.ravel(), comp_stride=case.n_points)
                   for k, v in case.fields.items())
    return Snapshot(0.0, 0, 0, (SemBlock(case.n_elements, case.x, case.y, case.z, fields=fields,
                                         global_ids=case.global_ids() if gid else None),))


@pytest.mark.parametrize("nel", [(2, 2, 2), (4, 3, 3)])
def test_dssum_matches_oracle(ctx, nel):
    case = synth.rbc_cylinder(nel=nel)
    da = SemDataAdaptor(ctx)
    da.initialize(_snapshot(case))
    rng = np.random.default_rng(1)
    v = rng.standard_normal(case.n_points)
    d = DeviceArray.empty(ctx, (v.size,), np.float64)
    d.upload(v)
    ctx.dssum(d)
    got = d.to_host()
    exp = O.dssum(case.global_ids(), v)
    assert np.array_equal(got.view(np.uint64), exp.view(np.uint64))
    # C0: every copy of an id holds the same value
    gid = case.global_ids()
    o = np.argsort(gid, kind="stable")
    first = np.flatnonzero(np.r_[True, gid[o][1:] != gid[o][:-1]])
    assert np.array_equal(got[o], np.repeat(got[o][first], np.diff(np.r_[first, got.size])))


def test_dssum_needs_global_ids(ctx):
    case = synth.box(nel=(1, 1, 2))
    da = SemDataAdaptor(ctx)
    da.initialize(_snapshot(case, gid=False))
    d = DeviceArray.empty(ctx, (case.n_points,), np.float64)
    with pytest.raises(RuntimeError, match="global_ids"):
        ctx.dssum(d)


def test_continuous_pipeline_equals_oracle_on_averaged_q(ctx):
    case = synth.rbc_cylinder(nel=(4, 4, 3))
    da = SemDataAdaptor(ctx)
    da.initialize(_snapshot(case))
    pipe = Pipeline(surfaces=(Surface("iso", "Q", 1.0), Surface("iso", "temperature", 0.5)),
                    color_field="Q", emit_meta=True, continuous=True)
    res = InsituAnalysis(pipe).execute(da, depth=True)
    cf = O.CaseFields(case.x, case.y, case.z, case.fields)
    q, _, _, _ = O.derived(cf)
    qc = O.dssum(case.global_ids(), q)
    cf2 = O.CaseFields(case.x, case.y, case.z, {**case.fields, "Qc": qc[None]})
    tri, meta, (cmin, cmax) = O.mc(cf2, [("iso", "Qc", 1.0), ("iso", "temperature", 0.5)], "Qc")
    gt, gm = ctx.triangles(with_meta=True)
    assert res.report.n_triangles == len(tri)
    assert np.array_equal(gm, meta)
    assert np.array_equal(gt.view(np.uint32), tri.view(np.uint32))
    assert res.report.range == (cmin, cmax)
    z = O.raster(tri, res.view, pipe.width, pipe.height)
    rgba, dep = O.resolve(z, pipe.width, pipe.height, cmin, cmax)
    assert np.array_equal(res.rgba, rgba) and np.array_equal(res.depth.view(np.uint32), dep.view(np.uint32))
    # without averaging, the element-local Q differs on shared nodes and the
    # triangles move (the surface cracks along element faces)
    assert not np.array_equal(qc, q)
    InsituAnalysis(Pipeline(**{**pipe.__dict__, "continuous": False})).execute(da)
    gt2 = ctx.triangles()
    assert len(gt2) != len(gt) or not np.array_equal(gt2.view(np.uint32), gt.view(np.uint32))


def _irregular_ids(n, rng):
    """Global ids with runs of 1..12 copies, some far longer (serial path of the
    one-pass kernel), scattered over the local positions."""
    lens = list(rng.integers(1, 13, size=n))
    lens[3] = 40
    lens[10] = 300
    ids = np.repeat(np.arange(len(lens), dtype=np.int64), lens)[:n]
    rng.shuffle(ids)
    return ids * 7 + 3                       # sparse, non-contiguous ids


@pytest.mark.parametrize("two_pass", [False, True])
@pytest.mark.parametrize("kind", ["irregular", "one_id", "all_distinct", "pairs_on_warp_edges"])
def test_dssum_irregular_runs_match_oracle(ctx, monkeypatch, kind, two_pass):
    """One-rank DSSUM (one-pass warp kernel, and the two-pass sum/scatter
    kernels) on id layouts that stress the warp windows: runs of 1..300
    copies in random positions, a single id shared by every copy, no sharing
    at all, and pairs straddling every warp boundary."""
    import torch

    if two_pass:
        monkeypatch.setenv("NKB_DSSUM_TWO_PASS", "1")
    case = synth.box(nel=(3, 2, 2))
    n = case.n_points
    rng = np.random.default_rng(7)
    if kind == "irregular":
        gid = _irregular_ids(n, rng)
    elif kind == "one_id":
        gid = np.full(n, 5, dtype=np.int64)
    elif kind == "all_distinct":
        gid = rng.permutation(n).astype(np.int64)
    else:
        gid = (np.arange(n, dtype=np.int64) + 1) // 2      # runs [0], [1,2], [3,4], ...: every 32nd pair splits
    da = SemDataAdaptor(ctx)
    da.initialize(_snapshot(case, gid=False))
    ctx.mesh_set_global_ids(torch.from_numpy(gid).cuda())
    v = rng.standard_normal(n)
    d = DeviceArray.empty(ctx, (n,), np.float64)
    d.upload(v)
    ctx.dssum(d)
    got = d.to_host()
    exp = O.dssum(gid, v)
    assert np.array_equal(got.view(np.uint64), exp.view(np.uint64))
