"""BASELINE.json's full sizes, checked through size-independent properties
(the oracle is too slow there; C2 at full size is compared with the oracle
directly in test_gpu_parity.py):

* C3 (250,000 elements): the geometry-cached and recomputing kernels give
  the same triangle count, colour range and image bit for bit; the FAST
  (per-CTA regions) and ORDERED (count/scan/emit) modes emit the same
  triangle multiset;
* C4 (1,048,576 elements, 537M GLL points, 6.5M triangles): FAST vs
  ORDERED triangle multisets and identical images;
* C3 and C4: element windows of the full-size run (first, middle, last,
  seeded, and for C4 the layers the slice plane cuts) against the C oracle
  on host copies of the same device bytes -- triangles and case words
  bit-exact (elements are independent, so a window needs only its own data).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _setup(name):
    from paper_2312_09888_b200 import synth_device
    from paper_2312_09888_b200.adaptor import SemDataAdaptor
    from paper_2312_09888_b200.analysis import pipeline_from_params
    from paper_2312_09888_b200.context import Context
    from paper_2312_09888_b200.data_model import POINT, FieldArray, SemBlock, Snapshot

    case = synth_device.make_case(name, 0, 1, device="cuda:0")
    ctx = Context(0)
    da = SemDataAdaptor(ctx)
    fields = tuple(FieldArray(k, POINT, v.shape[0], v.reshape(-1), comp_stride=case.n_points)
                   for k, v in case.fields.items())
    da.initialize(Snapshot(0.0, 0, 0, (SemBlock(case.n_elements, case.x, case.y, case.z, fields=fields),)))
    pipe = pipeline_from_params({**case.params, "width": "512", "height": "512"})
    da._case = case                      # the device arrays the adaptor borrows
    return ctx, da, pipe


def _sorted_rows(t):
    v = np.ascontiguousarray(t).reshape(len(t), -1).view(np.uint32)
    return v[np.lexsort(v.T[::-1])]


def test_c3_cached_uncached_fast_ordered():
    from dataclasses import replace

    from paper_2312_09888_b200.analysis import InsituAnalysis

    ctx, da, pipe = _setup("c3")
    an = InsituAnalysis(pipe)
    a = an.execute(da, depth=True)
    fast = ctx.triangles()
    ctx.set_geometry_cache(False)
    b = an.execute(da, depth=True)
    ctx.set_geometry_cache(True)
    assert a.report.n_triangles == b.report.n_triangles > 1000
    assert a.report.range == b.report.range
    assert np.array_equal(a.rgba, b.rgba) and np.array_equal(a.depth.view(np.uint32), b.depth.view(np.uint32))
    o = InsituAnalysis(replace(pipe, emit_meta=True)).execute(da)
    ordered, meta = ctx.triangles(with_meta=True)
    assert o.report.n_triangles == a.report.n_triangles
    assert np.array_equal(_sorted_rows(fast), _sorted_rows(ordered))
    assert np.all(np.diff(meta.astype(np.int64) >> 32) >= 0)          # element-major order
    assert np.array_equal(o.rgba, a.rgba)
    ctx.close()


def test_c4_fast_vs_ordered():
    from dataclasses import replace

    from paper_2312_09888_b200.analysis import InsituAnalysis

    ctx, da, pipe = _setup("c4")
    a = InsituAnalysis(pipe).execute(da, depth=True)
    fast = ctx.triangles()
    o = InsituAnalysis(replace(pipe, emit_meta=True)).execute(da, depth=True)
    ordered = ctx.triangles()
    assert a.report.n_triangles == o.report.n_triangles > 1_000_000
    assert np.array_equal(_sorted_rows(fast), _sorted_rows(ordered))
    assert np.array_equal(a.rgba, o.rgba) and np.array_equal(a.depth.view(np.uint32), o.depth.view(np.uint32))
    ctx.close()


def _window_oracle(ctx, da, pipe, case_dev, windows, around_triangles=0, w=48, seed=0):
    """Ordered-mode GPU triangles + meta of the full mesh against the C
    oracle run on host copies of element windows [e0, e1): every window's
    triangles and (element, cell, surface, case) words must be identical
    (elements are independent, so the oracle needs only the window)."""
    from dataclasses import replace

    from oracle import oracle as O
    from paper_2312_09888_b200.analysis import InsituAnalysis

    res = InsituAnalysis(replace(pipe, emit_meta=True)).execute(da)
    tri, meta = ctx.triangles(with_meta=True)
    assert res.report.n_triangles == len(tri)
    elem = (meta >> np.uint64(32)).astype(np.int64)
    if around_triangles:                 # windows centred on seeded elements that emit triangles
        rng = np.random.default_rng(seed)
        E = case_dev.n_elements
        for c in rng.choice(np.unique(elem), size=around_triangles, replace=False):
            s0 = int(min(max(c - w // 2, 0), E - w))
            windows = list(windows) + [(s0, s0 + w)]
    surf = [("iso", s.field, s.value) if s.kind == "iso" else ("slice", s.normal, s.value) for s in pipe.surfaces]
    checked = 0
    for e0, e1 in windows:
        n0, n1 = e0 * 512, e1 * 512
        cf = O.CaseFields(case_dev.x[n0:n1].cpu().numpy(), case_dev.y[n0:n1].cpu().numpy(),
                          case_dev.z[n0:n1].cpu().numpy(),
                          {k: v[:, n0:n1].contiguous().cpu().numpy() for k, v in case_dev.fields.items()})
        otri, ometa, _ = O.mc(cf, surf, pipe.color_field)
        sel = (elem >= e0) & (elem < e1)
        gmeta = meta[sel] - (np.uint64(e0) << np.uint64(32))
        assert np.array_equal(gmeta, ometa), f"window [{e0}, {e1}): case words differ"
        assert np.array_equal(tri[sel].view(np.uint32), otri.view(np.uint32)), f"window [{e0}, {e1}): vertices differ"
        checked += len(otri)
    return checked


def _windows(E, w=48, seed=0):
    rng = np.random.default_rng(seed)
    starts = [0, E // 2 - w // 2, E - w] + [int(s) for s in rng.integers(0, E - w, size=3)]
    return [(s, s + w) for s in starts]


def test_c3_full_size_element_windows_match_oracle():
    """C3 at full size (250,000 elements, Q iso coloured by |w|): windows of 48
    elements (first, middle, last, three seeded, four centred on seeded
    triangle-emitting elements) bit-exact with the oracle."""
    ctx, da, pipe = _setup("c3")
    case = da._case
    n = _window_oracle(ctx, da, pipe, case, _windows(case.n_elements, seed=3), around_triangles=4, seed=3)
    assert n > 0
    ctx.close()


def test_c4_full_size_element_windows_match_oracle():
    """C4 at full size (1,048,576 elements: |u| iso + z=0.5 slice, K1s): six
    windows bit-exact with the oracle, plus windows on the slice plane."""
    ctx, da, pipe = _setup("c4")
    case = da._case
    E = case.n_elements
    wins = _windows(E, seed=4) + [(E // 2, E // 2 + 48), (E // 2 - 48, E // 2)]   # the z = 0.5 slice lies on the element layer boundary at E/2
    n = _window_oracle(ctx, da, pipe, case, wins, around_triangles=4, seed=4)
    assert n > 0
    ctx.close()
