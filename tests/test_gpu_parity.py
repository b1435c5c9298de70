"""GPU parity: the CUDA path, called through the C ABI (Context -> ctypes ->
libnekb200), against the CPU oracle on identical synthetic SEM fields.

Bar (north star): connectivity, case indices, triangle counts bit-exact;
derived fields bit-exact with the oracle (which is itself within 1e-12 of an
independent numpy formulation, tests/test_oracle.py); images and depth
bit-exact (per-pixel tolerance 0).
"""
import math
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2312_09888_b200 import synth
from paper_2312_09888_b200.adaptor import SemDataAdaptor
from paper_2312_09888_b200.analysis import InsituAnalysis, Pipeline, Surface, ortho_view
from paper_2312_09888_b200.data_model import POINT, FieldArray, SemBlock, Snapshot

pytestmark = pytest.mark.gpu


def _snapshot(case, step=0, aos=False):
    fields = []
    for k, v in case.fields.items():
        if aos and v.shape[0] > 1:
            fields.append(FieldArray(k, POINT, v.shape[0], v.T.ravel()))        # reference AoS layout
        else:
            fields.append(FieldArray(k, POINT, v.shape[0], v.ravel(), comp_stride=case.n_points))
    blk = SemBlock(case.n_elements, case.x, case.y, case.z, fields=tuple(fields),
                   element_offset=case.e0, n_elements_global=case.n_elements_global)
    return Snapshot(0.0, step, 0, (blk,))


def _orc_surfaces(pipe):
    return [("iso", s.field, s.value) if s.kind == "iso" else ("slice", s.normal, s.value) for s in pipe.surfaces]


def _run(ctx, case, pipe, aos=False):
    da = SemDataAdaptor(ctx)
    da.initialize(_snapshot(case, aos=aos))
    res = InsituAnalysis(pipe).execute(da, depth=True)
    return da, res


def _check_against_oracle(ctx, case, pipe, res, meta=True):
    cf = O.CaseFields(case.x, case.y, case.z, case.fields)
    tri, m, (cmin, cmax) = O.mc(cf, _orc_surfaces(pipe), pipe.color_field)
    assert res.report.n_triangles == len(tri)
    gt, gm = ctx.triangles(with_meta=True)
    if meta:
        assert np.array_equal(gm, m), "case indices / emission order differ"
    assert np.array_equal(gt.view(np.uint32), tri.view(np.uint32)), "triangle vertices differ"
    lo = cmin if pipe.vmin is None else pipe.vmin
    hi = cmax if pipe.vmax is None else pipe.vmax
    assert res.report.range == (lo, hi)
    z = O.raster(tri, res.view, pipe.width, pipe.height)
    rgba, dep = O.resolve(z, pipe.width, pipe.height, lo, hi, pipe.anchors, pipe.background)
    assert np.array_equal(res.rgba, rgba), f"{int(np.any(res.rgba != rgba, -1).sum())} pixels differ"
    assert np.array_equal(res.depth.view(np.uint32), dep.view(np.uint32))


BOX_PIPES = {
    "q_iso": Pipeline(surfaces=(Surface("iso", "Q", 0.5),), color_field="temperature"),
    "three_surfaces": Pipeline(surfaces=(Surface("iso", "Q", 0.5), Surface("iso", "temperature", 0.6),
                                         Surface("slice", value=0.9, normal=(0.3, 1.0, 0.2))),
                               color_field="temperature", view_dir=(30.0, 40.0)),
    "colour_q": Pipeline(surfaces=(Surface("iso", "temperature", 0.6),), color_field="Q", width=100, height=77),
    "colour_wmag": Pipeline(surfaces=(Surface("iso", "vorticity:mag", 1.0),), color_field="vorticity:mag"),
    "colour_umag_range": Pipeline(surfaces=(Surface("iso", "velocity:mag", 0.6),), color_field="velocity:mag",
                                  vmin=0.2, vmax=0.9),
    "custom_cmap_bg": Pipeline(surfaces=(Surface("slice", value=0.5, normal=(0, 0, 1)),
                                         Surface("slice", value=1.0, normal=(1, 0, 0))),
                               color_field="temperature", background=(10, 20, 30, 40),
                               anchors=((0.0, (0, 0, 0)), (0.3, (255, 0, 0)), (0.7, (0, 255, 0)),
                                        (1.0, (255, 255, 255))), view_dir=(-120.0, 10.0)),
    # K1g stages only the coordinates a slice normal uses: axis-aligned planes,
    # including planes through node coordinates (distances of exactly 0)
    "q_slice_y_on_nodes": Pipeline(surfaces=(Surface("iso", "Q", 0.5), Surface("slice", value=0.5, normal=(0, 1, 0))),
                                   color_field="temperature"),
    "q_slices_x_z": Pipeline(surfaces=(Surface("iso", "Q", 0.5), Surface("slice", value=0.25, normal=(1, 0, 0)),
                                       Surface("slice", value=0.5, normal=(0, 0, 1))),
                             color_field="Q", view_dir=(20.0, 60.0)),
    "q_slice_face": Pipeline(surfaces=(Surface("iso", "temperature", 0.6),
                                       Surface("slice", value=0.0, normal=(0, -1, 0))),
                             color_field="vorticity:mag"),
    # the same for K1s (no gradient): |u| iso + a slice through node coordinates
    "umag_slice_y_on_nodes": Pipeline(surfaces=(Surface("iso", "velocity:mag", 0.6),
                                                Surface("slice", value=0.5, normal=(0, 1, 0))),
                                      color_field="velocity:mag"),
    "four_surfaces": Pipeline(surfaces=(Surface("iso", "Q", -0.5), Surface("iso", "Q", 0.5),
                                        Surface("iso", "temperature", 0.2),
                                        Surface("slice", value=0.7, normal=(1, 1, 1))),
                              color_field="Q", width=300, height=200),
    # the shapes K1g runs as compile-time node programs (fused.cu node_prog):
    # C2 (scalar iso + Q iso + slice, colour scalar), C3 (Q iso, colour |w|),
    # C1/C5 (Q iso, colour |u|); q_iso above is program 3
    "prog_c2": Pipeline(surfaces=(Surface("iso", "temperature", 0.6), Surface("iso", "Q", 0.5),
                                  Surface("slice", value=0.75, normal=(0, 1, 0))), color_field="temperature",
                        view_dir=(-60.0, 25.0)),
    "prog_c3": Pipeline(surfaces=(Surface("iso", "Q", 0.5),), color_field="vorticity:mag"),
    "prog_c1": Pipeline(surfaces=(Surface("iso", "Q", 0.5),), color_field="velocity:mag", view_dir=(35.0, 30.0)),
}


@pytest.mark.parametrize("name", list(BOX_PIPES))
def test_box_pipelines_bit_exact(ctx_geo, name):
    case = synth.box(nel=(4, 3, 3))
    pipe = Pipeline(**{**BOX_PIPES[name].__dict__, "emit_meta": True})
    _, res = _run(ctx_geo, case, pipe)
    _check_against_oracle(ctx_geo, case, pipe, res)


def _rows(t):
    return sorted(bytes(r) for r in np.ascontiguousarray(t).reshape(len(t), -1).view(np.uint8))


@pytest.mark.parametrize("name", ["three_surfaces", "four_surfaces"])
def test_fast_path_triangle_set_and_image(ctx, name):
    """Unordered fast path (atomic slot allocation): same triangle multiset,
    identical image (order-independent raster)."""
    case = synth.box(nel=(4, 3, 3))
    pipe = BOX_PIPES[name]
    _, res = _run(ctx, case, pipe)
    cf = O.CaseFields(case.x, case.y, case.z, case.fields)
    tri, _, (cmin, cmax) = O.mc(cf, _orc_surfaces(pipe), pipe.color_field)
    gt = ctx.triangles()
    assert len(gt) == len(tri) and _rows(gt) == _rows(tri)
    z = O.raster(tri, res.view, pipe.width, pipe.height)
    rgba, _ = O.resolve(z, pipe.width, pipe.height, cmin, cmax)
    assert np.array_equal(res.rgba, rgba)


def test_taylor_green_c1_bit_exact(ctx_geo):
    case = synth.taylor_green()
    pipe = Pipeline(surfaces=(Surface("iso", "Q", 0.1),), color_field="velocity:mag", width=256, height=256,
                    view_dir=(35.0, 30.0), emit_meta=True)
    _, res = _run(ctx_geo, case, pipe)
    _check_against_oracle(ctx_geo, case, pipe, res)


def test_aos_host_velocity_layout(ctx):
    """Host velocity in the reference's component-fastest AoS layout (data_model.py:8-14)."""
    case = synth.box(nel=(2, 2, 2))
    pipe = Pipeline(surfaces=(Surface("iso", "Q", 0.5),), color_field="velocity:mag", emit_meta=True)
    _, res = _run(ctx, case, pipe, aos=True)
    _check_against_oracle(ctx, case, pipe, res)


def test_c2_full_config_matches_oracle(ctx):
    """BASELINE configs[1] at full size (32,768 elements, 16.8M GLL points)."""
    case = synth.make_case("c2")
    from paper_2312_09888_b200.analysis import pipeline_from_params

    pipe = pipeline_from_params({**case.params, "width": "512", "height": "512"})
    _, res = _run(ctx, case, pipe)
    cf = O.CaseFields(case.x, case.y, case.z, case.fields)
    rgba, dep, ntri, rng = O.pipeline_mt(cf, _orc_surfaces(pipe), pipe.color_field, res.view, 512, 512,
                                         os.cpu_count() or 8)
    assert res.report.n_triangles == ntri
    assert res.report.range == rng
    assert np.array_equal(res.rgba, rgba)
    assert np.array_equal(res.depth.view(np.uint32), dep.view(np.uint32))


def test_triangle_buffer_growth_reruns_deterministically(ctx):
    case = synth.box(nel=(4, 4, 4))
    rng = np.random.default_rng(5)
    noisy = rng.standard_normal(case.n_points)            # ~1 triangle per cell -> > initial capacity
    case.fields["noise"] = noisy[None]
    pipe = Pipeline(surfaces=(Surface("iso", "noise", 0.0), Surface("iso", "noise", 0.5),
                              Surface("iso", "noise", -0.5), Surface("iso", "noise", 1.0)),
                    color_field="noise", emit_meta=True)
    from paper_2312_09888_b200.context import Context

    fresh = Context(0)          # new context: initial capacity max(65536, 16 E)
    _, res = _run(fresh, case, pipe)
    assert res.report.n_triangles > 65536 and res.report.reran
    _check_against_oracle(fresh, case, pipe, res)
    _, res2 = _run(fresh, case, pipe)
    assert not res2.report.reran and np.array_equal(res.rgba, res2.rgba)
    fresh.close()


def test_fast_path_region_overflow_reruns(ctx):
    """FAST mode (per-CTA triangle regions): a region that overflows triggers
    one re-run with larger regions; image and triangle multiset still exact."""
    case = synth.box(nel=(4, 4, 4))
    rng = np.random.default_rng(6)
    case.fields["noise"] = rng.standard_normal(case.n_points)[None]
    pipe = Pipeline(surfaces=(Surface("iso", "noise", 0.0), Surface("iso", "noise", 0.7)),
                    color_field="noise")
    from paper_2312_09888_b200.context import Context

    fresh = Context(0)
    _, res = _run(fresh, case, pipe)
    assert res.report.reran
    cf = O.CaseFields(case.x, case.y, case.z, case.fields)
    tri, _, (cmin, cmax) = O.mc(cf, _orc_surfaces(pipe), pipe.color_field)
    gt = fresh.triangles()
    assert len(gt) == len(tri) == res.report.n_triangles and _rows(gt) == _rows(tri)
    z = O.raster(tri, res.view, pipe.width, pipe.height)
    rgba, _ = O.resolve(z, pipe.width, pipe.height, cmin, cmax)
    assert np.array_equal(res.rgba, rgba)
    fresh.close()


def test_no_surfaces_gives_background(ctx):
    case = synth.box(nel=(2, 1, 1))
    pipe = Pipeline(surfaces=(), color_field="temperature", width=16, height=8, background=(1, 2, 3, 4))
    _, res = _run(ctx, case, pipe)
    assert res.report.n_triangles == 0
    assert (res.rgba.reshape(-1, 4) == [1, 2, 3, 4]).all() and np.isinf(res.depth).all()


def test_zero_elements_rank(ctx):
    """A rank that owns no elements (E = 0) still executes (empty partition)."""
    case = synth.box(0, 0, nel=(2, 2, 2))
    pipe = Pipeline(surfaces=(Surface("iso", "Q", 0.5),), color_field="temperature", width=8, height=8,
                    view=tuple(float(v) for v in ortho_view((0, 2, 0, 1.5, 0, 1), 8, 8)))
    _, res = _run(ctx, case, pipe)
    assert res.report.n_triangles == 0 and (res.rgba[..., 3] == 0).all()


def test_repeat_is_deterministic(ctx):
    case = synth.box(nel=(3, 3, 3))
    pipe = BOX_PIPES["three_surfaces"]
    da, r1 = _run(ctx, case, pipe)
    r2 = InsituAnalysis(pipe).execute(da, depth=True)
    assert np.array_equal(r1.rgba, r2.rgba) and np.array_equal(r1.depth, r2.depth)


# ------------------------------------------------------------- geometry cache


def _ro(a):
    a = np.array(a)
    a.flags.writeable = False
    return a


def test_static_mesh_reuses_geometry_cache(ctx):
    """Same read-only coordinate arrays step after step (static NekRS mesh):
    the cache is built once and reused; every step stays bit-exact."""
    case = synth.box(nel=(3, 3, 2))
    case.x, case.y, case.z = _ro(case.x), _ro(case.y), _ro(case.z)
    pipe = Pipeline(surfaces=(Surface("iso", "Q", 0.5),), color_field="vorticity:mag", emit_meta=True,
                    timing=True)
    da = SemDataAdaptor(ctx)
    an = InsituAnalysis(pipe)
    da.initialize(_snapshot(case))
    r1 = an.execute(da, depth=True)
    assert r1.report.geometry_cached
    h2d_first = da.h2d_bytes
    rng = np.random.default_rng(3)
    case.fields["velocity"] = case.fields["velocity"] + 0.1 * rng.standard_normal(case.fields["velocity"].shape)
    da.initialize(_snapshot(case, step=1))
    r2 = an.execute(da, depth=True)
    assert r2.report.geometry_cached and r2.report.ms_geometry == 0.0
    assert da.h2d_bytes == h2d_first - 3 * 8 * case.n_points         # coordinates not re-sent
    _check_against_oracle(ctx, case, pipe, r2)


def test_moving_mesh_rebuilds_geometry_cache(ctx):
    """New coordinates (host arrays) or in-place edits of device coordinates
    followed by mesh_modified() give the new mesh's exact results."""
    import torch

    case = synth.box(nel=(3, 2, 2))
    pipe = Pipeline(surfaces=(Surface("iso", "Q", 0.5),), color_field="temperature", emit_meta=True)
    da = SemDataAdaptor(ctx)
    an = InsituAnalysis(pipe)
    da.initialize(_snapshot(case))
    an.execute(da, depth=True)
    # host: deform the mesh, new arrays
    case.x = case.x + 0.05 * np.sin(3.0 * case.y)
    da.initialize(_snapshot(case, step=1))
    _check_against_oracle(ctx, case, pipe, an.execute(da, depth=True))
    # device arrays edited in place
    dev = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (case.x, case.y, case.z)]
    flds = tuple(FieldArray(k, POINT, v.shape[0], v.ravel(), comp_stride=case.n_points)
                 for k, v in case.fields.items())
    blk = lambda: Snapshot(0.0, 2, 0, (SemBlock(case.n_elements, *dev, fields=flds),))
    da.initialize(blk())
    an.execute(da, depth=True)
    case.z = case.z + 0.03 * np.cos(2.0 * case.x)
    dev[2].copy_(torch.from_numpy(case.z))
    da.initialize(blk())
    da.mesh_modified()
    _check_against_oracle(ctx, case, pipe, an.execute(da, depth=True))


def test_geometry_cache_layouts(ctx):
    """Extruded meshes (boxes, the curved C2-style cylinder) keep the compact
    cache (264 doubles per element); a mesh whose z varies in-plane falls
    back to the full 9 x 512 layout.  Compact, full and recomputed geometry
    give the oracle's results bit for bit."""
    pipe = Pipeline(surfaces=(Surface("iso", "Q", 0.5), Surface("slice", value=0.0, normal=(0, 1, 0))),
                    color_field="vorticity:mag", emit_meta=True)
    cyl = synth.rbc_cylinder(nel=(4, 4, 3))
    twisted = synth.box(nel=(3, 2, 2))
    twisted.z = twisted.z + 0.03 * np.cos(2.0 * twisted.x)          # z depends on (i, j): not extruded
    for case, layout in ((synth.box(nel=(3, 3, 2)), "compact"), (cyl, "compact"), (twisted, "full")):
        for mode, want in (("auto", layout), ("full", "full"), (False, "none")):
            ctx.set_geometry_cache(mode)
            da, res = _run(ctx, case, pipe)
            info = ctx.geometry_info()
            assert info["layout"] == want, (mode, info)
            if want == "compact":
                assert info["bytes"] == case.n_elements * 264 * 8
            elif want == "full":
                assert info["bytes"] == case.n_points * 72
            _check_against_oracle(ctx, case, pipe, res)
    ctx.set_geometry_cache(True)


# ---------------------------------------------------------------- DataAdaptor


def test_get_mesh_connectivity_and_points(ctx):
    case = synth.box(nel=(2, 2, 1))
    da = SemDataAdaptor(ctx)
    da.initialize(_snapshot(case))
    md = da.get_mesh_metadata()
    assert (md.n_elements, md.n_points, md.n_cells, md.cell_type) == (4, 2048, 1372, 12)
    g = da.get_mesh()
    conn = g.connectivity.to_host()
    e, a, b, c = np.meshgrid(np.arange(4), np.arange(7), np.arange(7), np.arange(7), indexing="ij")
    # cells ordered (e, c, b, a) with a fastest
    e, a, b, c = (v.transpose(0, 3, 2, 1).ravel() for v in (e, a, b, c))
    n0 = e * 512 + a + 8 * b + 64 * c
    expect = np.stack([n0, n0 + 1, n0 + 9, n0 + 8, n0 + 64, n0 + 65, n0 + 73, n0 + 72], axis=1)
    assert np.array_equal(conn, expect)
    assert np.array_equal(g.offsets.to_host(), 8 * np.arange(1373))
    assert (g.types.to_host() == 12).all()
    pts = g.points.to_host()
    assert np.array_equal(pts, np.stack([case.x, case.y, case.z], axis=1))


def test_add_array_exports_bit_exact(ctx_geo):
    ctx = ctx_geo
    case = synth.box(nel=(3, 2, 2))
    da = SemDataAdaptor(ctx)
    da.initialize(_snapshot(case))
    cf = O.CaseFields(case.x, case.y, case.z, case.fields)
    q, wm, vort, um = O.derived(cf)
    assert np.array_equal(da.add_array("mesh", POINT, "Q").values.to_host(), q)
    assert np.array_equal(da.add_array("mesh", POINT, "vorticity:mag").values.to_host(), wm)
    v = da.add_array("mesh", POINT, "vorticity")
    assert v.components == 3 and np.array_equal(v.values.to_host(), vort)
    assert np.array_equal(da.add_array("mesh", POINT, "velocity:mag").values.to_host(), um)
    vel = da.add_array("mesh", POINT, "velocity")
    assert np.array_equal(vel.values.to_host(), case.fields["velocity"].T.ravel())   # AoS
    x, y, z = case.x, case.y, case.z
    u = case.fields["velocity"]
    qn, _, _, g2 = O.derived_numpy(x, y, z, u[0], u[1], u[2])
    assert np.max(np.abs(q - qn)) <= 1e-12 * g2.max()


def test_errors_map_to_reference_exceptions(ctx):
    case = synth.box(nel=(1, 1, 1))
    da = SemDataAdaptor(ctx)
    da.initialize(_snapshot(case))
    an = InsituAnalysis(Pipeline(surfaces=(Surface("iso", "nope", 0.0),), color_field="temperature"))
    with pytest.raises(ValueError, match="no field named"):
        an.execute(da)
    an = InsituAnalysis(Pipeline(surfaces=(), color_field="velocity"))
    with pytest.raises(ValueError, match="components"):
        an.execute(da)
    an = InsituAnalysis(Pipeline(surfaces=(), color_field="temperature:grad"))
    with pytest.raises(ValueError, match="derived scalar"):
        an.execute(da)
    with pytest.raises(ValueError, match="order"):
        ctx.mesh_set(1, 0, 0, 0, order=5)


def test_abi_error_paths(ctx):
    """Argument and state errors of the newer entry points map to the
    reference's exception vocabulary (ValueError / RuntimeError)."""
    import ctypes as C

    from paper_2312_09888_b200 import _native as N
    from paper_2312_09888_b200.device import DeviceArray

    case = synth.box(nel=(1, 1, 1))
    da = SemDataAdaptor(ctx)
    da.initialize(_snapshot(case))
    d = DeviceArray.empty(ctx, (8,), np.float64)
    with pytest.raises(ValueError, match="segment shape"):
        ctx.stats([(d.ptr, 4, 0, 4)])
    with pytest.raises(ValueError, match="comp_stride"):
        ctx.stats([(d.ptr, 4, 2, 3)])
    n = C.c_int64()
    with pytest.raises(ValueError, match="too small"):
        N.call("nkb_encode_be", ctx.handle, b"POINTS", d.ptr, 8, C.byref(n), None)
    with pytest.raises(ValueError, match="no field named"):
        N.call("nkb_encode_be", ctx.handle, b"pressure", None, 0, C.byref(n), None)
    with pytest.raises(RuntimeError, match="communicator"):
        ctx.transit_gather(0)
    pipe = Pipeline(surfaces=(Surface("iso", "Q", 0.5),), color_field="temperature",
                    view=tuple([1.0] * 12) + (0.0, 0.0, float("nan"), 1.0))
    with pytest.raises(ValueError, match="perspective row"):
        InsituAnalysis(pipe).execute(da)
    with pytest.raises(ValueError, match="12 values"):
        InsituAnalysis(Pipeline(view=(1.0,) * 13)).execute(da)


NOGRAD_PIPES = {
    "umag_iso_umag_colour": Pipeline(surfaces=(Surface("iso", "velocity:mag", 0.6),
                                               Surface("slice", value=0.5, normal=(0, 0, 1))),
                                     color_field="velocity:mag"),
    "scalar_iso_two_slices": Pipeline(surfaces=(Surface("iso", "temperature", 0.4),
                                                Surface("slice", value=0.9, normal=(0.3, 1.0, 0.2)),
                                                Surface("slice", value=1.0, normal=(1, 0, 0))),
                                      color_field="temperature", width=120, height=90),
    "four_no_grad": Pipeline(surfaces=(Surface("iso", "temperature", 0.2), Surface("iso", "temperature", 0.7),
                                       Surface("iso", "velocity:mag", 0.5),
                                       Surface("slice", value=0.7, normal=(1, 1, 1))),
                             color_field="temperature"),
}


@pytest.mark.parametrize("name", list(NOGRAD_PIPES))
def test_stream_pass_matches_fused_pass_and_oracle(ctx, name, monkeypatch):
    """Pipelines without a velocity gradient run the warp-per-element pass
    (stream.cu, report.surface_pass == 1); NKB_STREAM=0 forces K1.  Both
    give the oracle's triangles (ordered: same list and case words; fast:
    same multiset) and identical images."""
    case = synth.box(nel=(4, 3, 3))
    out = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("NKB_STREAM", mode)
        pipe = Pipeline(**{**NOGRAD_PIPES[name].__dict__, "emit_meta": True})
        _, res = _run(ctx, case, pipe)
        assert res.report.surface_pass == int(mode)
        _check_against_oracle(ctx, case, pipe, res)
        _, fast = _run(ctx, case, NOGRAD_PIPES[name])
        assert fast.report.surface_pass == int(mode)
        out[mode] = (_rows(ctx.triangles()), fast.rgba.copy(), fast.report.range)
    assert out["1"][0] == out["0"][0]
    assert np.array_equal(out["1"][1], out["0"][1]) and out["1"][2] == out["0"][2]


def test_gradient_pipelines_use_fused_pass(ctx):
    """Gradient pipelines run K1 (uncached geometry) or K1g (cached geometry,
    two CTAs per SM, report.surface_pass == 2; NKB_FUSED2=0 forces K1)."""
    case = synth.box(nel=(2, 2, 2))
    ctx.set_geometry_cache(False)
    _, res = _run(ctx, case, BOX_PIPES["q_iso"])
    assert res.report.surface_pass == 0
    ctx.set_geometry_cache(True)
    _, res = _run(ctx, case, BOX_PIPES["q_iso"])
    assert res.report.surface_pass == 2


@pytest.mark.parametrize("geo", ["auto", "full"])
@pytest.mark.parametrize("name", ["q_iso", "three_surfaces", "colour_wmag", "four_surfaces"])
def test_two_cta_gradient_pass_matches_k1_and_oracle(ctx, name, geo, monkeypatch):
    """K1g (two 256-thread CTAs per SM) against K1 and the oracle: ordered
    triangles and case words, fast-path multisets, images and ranges; with
    the compact (extruded box) and the full geometry cache.  K1g stages up to
    7 inputs (6 with the compact cache); beyond that K1 runs."""
    case = synth.box(nel=(5, 4, 3))
    ctx.set_geometry_cache(geo)
    staged = {"q_iso": 4, "three_surfaces": 7, "colour_wmag": 3, "four_surfaces": 7}[name]
    fits = staged <= (6 if geo == "auto" else 7)
    out = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("NKB_FUSED2", mode)
        pipe = Pipeline(**{**BOX_PIPES[name].__dict__, "emit_meta": True})
        _, res = _run(ctx, case, pipe)
        assert res.report.surface_pass == (2 if (mode == "1" and fits) else 0)
        assert ctx.geometry_info()["layout"] == ("compact" if geo == "auto" else "full")
        _check_against_oracle(ctx, case, pipe, res)
        _, fast = _run(ctx, case, BOX_PIPES[name])
        out[mode] = (_rows(ctx.triangles()), fast.rgba.copy(), fast.report.range)
    assert out["1"][0] == out["0"][0]
    assert np.array_equal(out["1"][1], out["0"][1]) and out["1"][2] == out["0"][2]
    ctx.set_geometry_cache(True)


def test_large_triangles_raster_bit_exact(ctx):
    """A coarse mesh drawn big: triangles span hundreds of pixels (long
    per-thread pixel walks in K2, many atomicMin collisions between
    overlapping triangles); image and depth equal the oracle's."""
    case = synth.box(nel=(2, 2, 2))
    pipe = Pipeline(surfaces=(Surface("iso", "temperature", 0.45), Surface("slice", value=0.8, normal=(1, 0.2, 0))),
                    color_field="temperature", width=640, height=480, emit_meta=True)
    _, res = _run(ctx, case, pipe)
    tri = ctx.triangles()
    assert len(tri) > 0
    _check_against_oracle(ctx, case, pipe, res)


@pytest.mark.parametrize("name", ["prog_c2", "prog_c3", "prog_c1", "q_iso"])
def test_node_programs_equal_generic_dispatch(ctx, name, monkeypatch):
    """Compile-time node programs (K1g) against the generic runtime dispatch
    (NKB_NODE_PROGS=0): identical ordered triangles, case words and images."""
    case = synth.rbc_cylinder(nel=(4, 4, 4))
    ctx.set_geometry_cache(True)
    out = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("NKB_NODE_PROGS", mode)
        pipe = Pipeline(**{**BOX_PIPES[name].__dict__, "emit_meta": True})
        _, res = _run(ctx, case, pipe)
        assert res.report.surface_pass == 2
        _check_against_oracle(ctx, case, pipe, res)
        out[mode] = (ctx.triangles(with_meta=True), res.rgba.copy(), res.report.range)
    assert np.array_equal(out["1"][0][1], out["0"][0][1])
    assert np.array_equal(out["1"][0][0].view(np.uint32), out["0"][0][0].view(np.uint32))
    assert np.array_equal(out["1"][1], out["0"][1]) and out["1"][2] == out["0"][2]


def test_stream_node_program_equals_generic(ctx, monkeypatch):
    """K1s node program 1 (|u| iso + slice, colour |u|: the C4 shape) against
    the generic K1s dispatch and the oracle."""
    case = synth.box(nel=(4, 3, 3))
    out = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("NKB_NODE_PROGS", mode)
        pipe = Pipeline(**{**NOGRAD_PIPES["umag_iso_umag_colour"].__dict__, "emit_meta": True})
        _, res = _run(ctx, case, pipe)
        assert res.report.surface_pass == 1
        _check_against_oracle(ctx, case, pipe, res)
        out[mode] = (ctx.triangles(with_meta=True), res.rgba.copy(), res.report.range)
    assert np.array_equal(out["1"][0][1], out["0"][0][1])
    assert np.array_equal(out["1"][0][0].view(np.uint32), out["0"][0][0].view(np.uint32))
    assert np.array_equal(out["1"][1], out["0"][1]) and out["1"][2] == out["0"][2]


# ------------------------------------------------------------ stream-ordered execute


def test_execute_async_matches_execute(ctx):
    """nkb_execute_async x 3 then nkb_execute_wait: the same image, triangle
    set and report as the synchronous execute."""
    case = synth.rbc_cylinder(nel=(4, 4, 4))
    pipe = BOX_PIPES["prog_c2"]
    da, ref = _run(ctx, case, pipe)
    tri_ref = _rows(ctx.triangles())
    an = InsituAnalysis(pipe)
    for _ in range(3):
        an.execute_async(da)
    rep = an.wait()
    assert not rep.overflowed and rep.n_triangles == ref.report.n_triangles
    assert rep.range == ref.report.range and rep.surface_pass == ref.report.surface_pass
    rgba, dep = ctx.image(pipe.width, pipe.height, depth=True)
    assert np.array_equal(rgba, ref.rgba) and np.array_equal(dep.view(np.uint32), ref.depth.view(np.uint32))
    assert _rows(ctx.triangles()) == tri_ref


def test_execute_async_overflow_is_reported_then_grown(monkeypatch):
    """An async step cannot re-run: with a tiny initial triangle buffer the
    first step reports overflowed=True, the buffer grows, and the next async
    step is complete (equal to the synchronous result)."""
    from paper_2312_09888_b200.context import Context

    monkeypatch.setenv("NKB_TRI_CAP0", "64")
    c = Context(0)
    case = synth.box(nel=(3, 3, 2))
    pipe = BOX_PIPES["three_surfaces"]
    da = SemDataAdaptor(c)
    da.initialize(_snapshot(case))
    an = InsituAnalysis(pipe)
    an.execute_async(da)
    r1 = an.wait()
    assert r1.overflowed and r1.tri_capacity > 64
    an.execute_async(da)
    r2 = an.wait()
    assert not r2.overflowed
    rgba = c.image(pipe.width, pipe.height)
    ref = InsituAnalysis(pipe).execute(da)
    assert ref.report.n_triangles == r2.n_triangles and np.array_equal(ref.rgba, rgba)
    with pytest.raises(RuntimeError, match="without a pending"):
        c.wait()
    an.execute_async(da)
    with pytest.raises(RuntimeError, match="pending"):
        c.execute(pipe.native(an.view_for(da)))
    c.wait()
    c.close()
