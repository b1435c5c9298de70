"""GPU stats sink against numpy -- the reference's own
arithmetic (StatsSink, sinks.py:381-386: vals.min(), vals.max(), vals.mean()
of the concatenated field values).  The mean is numpy's pairwise summation
re-done on the GPU, so every comparison is bit-exact."""
import numpy as np
import pytest

from paper_2312_09888_b200 import synth
from paper_2312_09888_b200.bridge import initialize, parse_config
from paper_2312_09888_b200.data_model import POINT, Block, FieldArray, SemBlock, Snapshot
from paper_2312_09888_b200.device import DeviceArray
from paper_2312_09888_b200.sinks import StatsSink

pytestmark = pytest.mark.gpu


def _bits(x):
    return np.float64(x).view(np.uint64)


def _check(got, vals):
    exp = (vals.min(), vals.max(), vals.mean())
    assert [_bits(g) for g in got] == [_bits(e) for e in exp], (got, exp)


def _dev(ctx, a):
    d = DeviceArray.empty(ctx, (a.size,), np.float64)
    d.upload(np.ascontiguousarray(a, dtype=np.float64))
    return d


@pytest.mark.parametrize("n", [1, 2, 7, 8, 9, 15, 16, 127, 128, 129, 255, 256, 1000, 8191, 8192, 8193,
                               32768, 32769, 65536 + 13, 100003, 1 << 20, 2500007])
def test_pairwise_mean_bit_exact(ctx, n):
    rng = np.random.default_rng(n)
    a = rng.standard_normal(n) * 10.0 ** rng.integers(-6, 7, n)
    d = _dev(ctx, a)
    _check(ctx.stats([(d.ptr, n, 1, n)]), a)


def test_large_array_many_chunks(ctx):
    """33.5M values: ~1000 chunks combined up the top of the tree."""
    n = 33_554_437
    rng = np.random.default_rng(7)
    a = rng.random(n) * 1e3 - 400.0
    d = _dev(ctx, a)
    _check(ctx.stats([(d.ptr, n, 1, n)]), a)


def test_soa_components_read_in_aos_order(ctx):
    """A 3-component SoA device field is reduced in the reference's AoS order."""
    npts = 70001
    rng = np.random.default_rng(3)
    soa = rng.standard_normal((3, npts)) * np.array([[1.0], [1e-3], [1e4]])
    d = _dev(ctx, soa.ravel())
    _check(ctx.stats([(d.ptr, npts, 3, npts)]), soa.T.ravel())


def test_segments_concatenate_in_order(ctx):
    rng = np.random.default_rng(11)
    parts = [rng.standard_normal(n) for n in (5, 300, 1, 40000, 129)]
    devs = [_dev(ctx, a) for a in parts]
    _check(ctx.stats([(d.ptr, a.size, 1, a.size) for d, a in zip(devs, parts)]), np.concatenate(parts))


def test_nan_and_empty(ctx):
    a = np.arange(1000, dtype=np.float64)
    a[517] = np.nan
    d = _dev(ctx, a)
    mn, mx, mean = ctx.stats([(d.ptr, a.size, 1, a.size)])
    assert np.isnan(mn) and np.isnan(mx) and np.isnan(mean)
    with pytest.raises(ValueError, match="zero-size"):
        ctx.stats([])


def _reference_rows(s):
    """sinks.py:381-386 verbatim in numpy (the reference's own arithmetic)."""
    rows = []
    for f in s.blocks[0].fields:
        vals = np.concatenate([b.field_named(f.name).values for b in s.blocks])
        rows.append(f"{s.step},{s.time:.17g},{f.name},{vals.min():.17g},{vals.max():.17g},{vals.mean():.17g}")
    return "\n".join(rows) + "\n"


def test_stats_sink_structured_rows_match_reference(tmp_path):
    rng = np.random.default_rng(5)
    blocks = []
    for k in range(3):        # x-tiled producer blocks
        ni = 17 + 4 * k
        npts = ni * 9
        fields = (FieldArray("temperature", POINT, 1, rng.random(npts)),
                  FieldArray("velocity", POINT, 3, rng.standard_normal(3 * npts)))
        blocks.append(Block((0.0, 0.0, 0.0), (0.1, 0.1, 1.0), (0, ni - 1, 0, 8, 0, 0), fields))
    sink = StatsSink({"path": str(tmp_path / "s" / "stats.csv")})
    total = 0
    for step in range(3):
        s = Snapshot(0.25 * step, step, 0, tuple(blocks))
        total += sink.consume(s)
    text = (tmp_path / "s" / "stats.csv").read_text()
    exp = "step,time,field,min,max,mean\n" + "".join(_reference_rows(Snapshot(0.25 * k, k, 0, tuple(blocks)))
                                                     for k in range(3))
    assert text == exp and total == len(exp) - len("step,time,field,min,max,mean\n")


def test_stats_sink_sem_snapshot_through_bridge(tmp_path):
    case = synth.box(nel=(3, 2, 2))
    vel = case.fields["velocity"]
    fields = (FieldArray("velocity", POINT, 3, vel.T.ravel()),
              FieldArray("temperature", POINT, 1, case.fields["temperature"].ravel()))
    blk = SemBlock(case.n_elements, case.x, case.y, case.z, fields=fields)
    br = initialize(parse_config(f'<sensei><analysis type="stats" path="{tmp_path}/st.csv" frequency="1"/></sensei>'))
    for step in range(2):
        reps = br.update(Snapshot(0.5 * step, step, 0, (blk,)))
        assert all(r.error is None for r in reps), reps
    lines = (tmp_path / "st.csv").read_text().splitlines()
    assert lines[0] == "step,time,field,min,max,mean" and len(lines) == 5
    for f, line in zip(fields, lines[1:3]):
        v = np.asarray(f.values)
        assert line == f"0,0,{f.name},{v.min():.17g},{v.max():.17g},{v.mean():.17g}"
