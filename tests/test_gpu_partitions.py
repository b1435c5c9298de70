"""R16 on ONE GPU: the sort-last composite kernels (p2p_composite_bulk_kernel,
the default, and p2p_composite_kernel) over
R in-process partition contexts, each owning a contiguous element range of
the mesh (the NekRS partition), must give the 1-partition
image bit for bit -- min over packed depth|colour keys is associative and
commutative, and the global colour range is the min/max of every
partition's range words.  The multi-process NVLink path (test_gpu_multi.py)
needs >= 2 GPUs; this runs the same kernel on the driver's one-GPU box."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2312_09888_b200 import synth
from paper_2312_09888_b200.adaptor import SemDataAdaptor
from paper_2312_09888_b200.analysis import InsituAnalysis, Pipeline, Surface, ortho_view
from paper_2312_09888_b200.context import Context
from paper_2312_09888_b200.data_model import POINT, FieldArray, SemBlock, Snapshot

pytestmark = pytest.mark.gpu


def _block(case, e0, e1):
    n0, n1 = e0 * 512, e1 * 512
    fields = tuple(FieldArray(k, POINT, v.shape[0], np.ascontiguousarray(v[:, n0:n1]).ravel(), comp_stride=n1 - n0)
                   for k, v in case.fields.items())
    return SemBlock(e1 - e0, case.x[n0:n1], case.y[n0:n1], case.z[n0:n1], fields=fields, element_offset=e0,
                    n_elements_global=case.n_elements)


def _pipe(case, W=192, H=160, **kw):
    b = (case.x.min(), case.x.max(), case.y.min(), case.y.max(), case.z.min(), case.z.max())
    view = ortho_view(b, W, H, -60.0, 25.0)
    return Pipeline(surfaces=(Surface("iso", "temperature", 0.5), Surface("iso", "Q", 1.0),
                              Surface("slice", value=0.0, normal=(0, 1, 0))),
                    color_field="temperature", width=W, height=H, view=view, composite=False, **kw)


@pytest.fixture(scope="module")
def cyl():
    return synth.rbc_cylinder(nel=(4, 4, 9))            # 144 elements: ragged splits for R = 5, 7


@pytest.fixture(scope="module")
def one(cyl):
    ctx = Context(0)
    pipe = _pipe(cyl)
    da = SemDataAdaptor(ctx)
    da.initialize(Snapshot(0.0, 0, 0, (_block(cyl, 0, cyl.n_elements),)))
    res = InsituAnalysis(pipe).execute(da, depth=True)
    yield res
    ctx.close()


def _composite(cyl, pipe, R, steps=1):
    parts = []
    for r in range(R):
        e0, e1 = synth.partition(cyl.n_elements, r, R)
        ctx = Context(0)
        da = SemDataAdaptor(ctx)
        da.initialize(Snapshot(0.0, 0, r, (_block(cyl, e0, e1),)))
        for _ in range(steps):            # one-GPU steps alternate two key buffers
            InsituAnalysis(pipe).execute(da, fetch_image=False)
        parts.append((ctx, da))
    root = parts[0][0]
    root.composite_partitions([c for c, _ in parts], pipe.native(pipe.view))
    rgba, depth = root.image(pipe.width, pipe.height, depth=True)
    for c, _ in parts:
        c.close()
    return rgba, depth


@pytest.mark.parametrize("R", [3, 8])
def test_bulk_and_load_kernels_agree_on_odd_bands(cyl, monkeypatch, R):
    """191 x 157 pixels: bands start and end on odd pixels, so the bulk-copy
    kernel's aligned tiles plus its end pixels must cover every band exactly;
    both composite kernels and the one-partition step agree bit for bit."""
    pipe = _pipe(cyl, W=191, H=157)
    ctx = Context(0)
    da = SemDataAdaptor(ctx)
    da.initialize(Snapshot(0.0, 0, 0, (_block(cyl, 0, cyl.n_elements),)))
    ref = InsituAnalysis(pipe).execute(da, depth=True)
    ctx.close()
    monkeypatch.setenv("NKB_COMPOSITE_BULK", "1")
    a_rgba, a_depth = _composite(cyl, pipe, R)
    c_rgba, c_depth = _composite(cyl, pipe, R, steps=2)   # the second key buffer (odd W*H: padded)
    monkeypatch.setenv("NKB_COMPOSITE_BULK", "0")
    b_rgba, b_depth = _composite(cyl, pipe, R)
    for rgba, depth in ((a_rgba, a_depth), (b_rgba, b_depth), (c_rgba, c_depth)):
        assert np.array_equal(rgba, ref.rgba)
        assert np.array_equal(depth.view(np.uint32), ref.depth.view(np.uint32))


@pytest.mark.parametrize("kernel", ["bulk", "loads"])
@pytest.mark.parametrize("R", [2, 3, 4, 5, 8])
def test_partition_composite_equals_one_partition(cyl, one, monkeypatch, R, kernel):
    monkeypatch.setenv("NKB_COMPOSITE_BULK", "1" if kernel == "bulk" else "0")
    pipe = _pipe(cyl)
    parts, ranges = [], []
    for r in range(R):
        e0, e1 = synth.partition(cyl.n_elements, r, R)
        ctx = Context(0)
        da = SemDataAdaptor(ctx)
        da.initialize(Snapshot(0.0, 0, r, (_block(cyl, e0, e1),)))
        rep = InsituAnalysis(pipe).execute(da, fetch_image=False).report
        parts.append((ctx, da))
        ranges.append(rep.data_range)
    root = parts[0][0]
    root.composite_partitions([c for c, _ in parts], pipe.native(pipe.view))
    rgba, depth = root.image(pipe.width, pipe.height, depth=True)
    assert np.array_equal(rgba, one.rgba), f"{int(np.any(rgba != one.rgba, -1).sum())} pixels differ"
    assert np.array_equal(depth.view(np.uint32), one.depth.view(np.uint32))
    # the global colour range the composite used = min/max over partitions
    assert min(r[0] for r in ranges) == one.report.range[0] and max(r[1] for r in ranges) == one.report.range[1]
    for c, _ in parts:
        c.close()


def test_partition_composite_matches_oracle(cyl):
    """The composited 4-partition image against the C oracle's full step."""
    pipe = _pipe(cyl)
    parts = []
    for r in range(4):
        e0, e1 = synth.partition(cyl.n_elements, r, 4)
        ctx = Context(0)
        da = SemDataAdaptor(ctx)
        da.initialize(Snapshot(0.0, 0, r, (_block(cyl, e0, e1),)))
        InsituAnalysis(pipe).execute(da, fetch_image=False)
        parts.append((ctx, da))
    root = parts[0][0]
    root.composite_partitions([c for c, _ in parts], pipe.native(pipe.view))
    rgba = root.image(pipe.width, pipe.height)
    cf = O.CaseFields(cyl.x, cyl.y, cyl.z, cyl.fields)
    surf = [("iso", "temperature", 0.5), ("iso", "Q", 1.0), ("slice", (0.0, 1.0, 0.0), 0.0)]
    ref, _, ntri, _ = O.pipeline_mt(cf, surf, "temperature", pipe.view, pipe.width, pipe.height, 4)
    assert ntri > 0
    assert np.array_equal(rgba, ref)
    for c, _ in parts:
        c.close()


def test_partition_composite_rejects_mismatched_image(cyl):
    pipe = _pipe(cyl)
    ctx = Context(0)
    da = SemDataAdaptor(ctx)
    da.initialize(Snapshot(0.0, 0, 0, (_block(cyl, 0, 8),)))
    InsituAnalysis(pipe).execute(da, fetch_image=False)
    other = _pipe(cyl, W=64, H=64)
    with pytest.raises(RuntimeError, match="key buffer"):
        ctx.composite_partitions([ctx], other.native(other.view))
    ctx.close()
