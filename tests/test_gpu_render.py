"""GPU drop-in for the reference's 2D pseudocolor renderer (sinks.render,
RenderSink) and the in situ sink behind the bridge, checked against golden
vectors made by the reference itself (tests/golden/make_golden.py) and the
oracle."""
import numpy as np
import pytest
from cases import RENDER_CASES, snapshot_arrays

from oracle import oracle as O
from paper_2312_09888_b200 import synth
from paper_2312_09888_b200.bridge import initialize, parse_config
from paper_2312_09888_b200.data_model import POINT, Block, FieldArray, SemBlock, Snapshot
from paper_2312_09888_b200.sinks import DEFAULT_COLORMAP, ImageRGB, RenderSink, render, write_ppm

pytestmark = pytest.mark.gpu

GOLD = np.load(f"{O.HERE}/../tests/golden/render.npz")


def _snapshot(seed, ni, nj, nk, nb, comps, step=3):
    blocks = []
    for temp, vel, ext in snapshot_arrays(seed, ni, nj, nk, nb, comps):
        f = (FieldArray("temperature", POINT, 1, temp), FieldArray("velocity", POINT, comps, vel))
        blocks.append(Block((ext[0] * 0.5, 0.0, 0.0), (0.5, 0.25, 1.0), ext, f))
    return Snapshot(0.0, step, 0, tuple(blocks))


@pytest.mark.parametrize("case", RENDER_CASES, ids=[f"case{c[0]}" for c in RENDER_CASES])
def test_render_matches_reference_golden(case):
    seed, ni, nj, nk, nb, comps, field, w, h, vmin, vmax = case
    img = render(_snapshot(seed, ni, nj, nk, nb, comps), field, DEFAULT_COLORMAP, w, h, vmin, vmax)
    assert np.array_equal(np.frombuffer(img.pixels, np.uint8), GOLD[f"case{seed}"])


@pytest.mark.parametrize("seed", range(6))
def test_render_random_shapes_match_oracle(seed):
    rng = np.random.default_rng(100 + seed)
    ni, nj, nb = int(rng.integers(1, 40)), int(rng.integers(1, 30)), int(rng.integers(1, 5))
    comps = int(rng.integers(1, 4))
    w, h = int(rng.integers(1, 300)), int(rng.integers(1, 200))
    s = _snapshot(seed, ni, nj, 1, nb, comps)
    for field in ("temperature", "velocity:mag"):
        img = render(s, field, DEFAULT_COLORMAP, w, h)
        mag = field.endswith(":mag")
        blocks = [(b.field_named("velocity" if mag else "temperature").values, ni) for b in s.blocks]
        px, _ = O.render_structured(blocks, nj, comps if mag else 1, int(mag), w, h)
        assert img.pixels == px


def test_render_reference_kats():
    # reference tests/test_sinks.py:229-246: row 0 is the top; degenerate range -> first anchor
    ni = nj = 4
    f = FieldArray("temperature", POINT, 1, np.repeat(np.arange(nj, dtype=float), ni))
    s = Snapshot(0.0, 0, 0, (Block((0, 0, 0), (1, 1, 1), (0, 3, 0, 3, 0, 0), (f,)),))
    px = np.frombuffer(render(s, "temperature", width=4, height=4).pixels, np.uint8).reshape(4, 4, 3)
    assert px[0, 0].tolist() == [180, 4, 38] and px[-1, 0].tolist() == [59, 76, 192]
    f = FieldArray("temperature", POINT, 1, np.full(16, 3.0))
    s = Snapshot(0.0, 0, 0, (Block((0, 0, 0), (1, 1, 1), (0, 3, 0, 3, 0, 0), (f,)),))
    assert render(s, "temperature", width=2, height=2).pixels == bytes([59, 76, 192]) * 4


def test_render_errors_match_reference():
    s = _snapshot(1, 3, 2, 1, 1, 2)
    with pytest.raises(ValueError, match="components"):
        render(s, "velocity")
    with pytest.raises(ValueError, match="derived"):
        render(s, "temperature:grad")
    with pytest.raises(KeyError):
        render(s, "pressure")


def test_render_sink_default_two_images(tmp_path):
    sink = RenderSink({"dir": str(tmp_path / "im"), "width": "16", "height": "16"})
    s = _snapshot(4, 5, 4, 1, 1, 2, step=7)
    n = sink.consume(s)
    files = sorted(p.name for p in (tmp_path / "im").glob("*.ppm"))
    assert files == ["step000007_temperature.ppm", "step000007_velocity_mag.ppm"]
    assert n == sum((tmp_path / "im" / f).stat().st_size for f in files) == 2 * (15 - 2 + 16 * 16 * 3)


def test_ppm_bytes_match_reference_golden(tmp_path):
    g = np.load(f"{O.HERE}/../tests/golden/ppm.npz")
    for (w, h) in ((1, 1), (3, 2), (256, 256)):
        rng = np.random.default_rng(w * 1000 + h)
        px = rng.integers(0, 256, size=3 * w * h, dtype=np.uint8).tobytes()
        n = write_ppm(ImageRGB(w, h, px), tmp_path / "a.ppm")
        raw = (tmp_path / "a.ppm").read_bytes()
        assert n == len(raw) and raw == g[f"ppm_{w}x{h}"].tobytes()


def test_insitu_sink_through_bridge(tmp_path):
    case = synth.box(nel=(3, 2, 2))
    doc = (f'<sensei><analysis type="insitu" frequency="2" dir="{tmp_path}/out" iso="Q=0.5;temperature=0.6" '
           f'slice="0.3,1,0.2,0.9" field="temperature" width="80" height="60" view="30,40"/>'
           f'<analysis type="null" frequency="1"/></sensei>')
    br = initialize(parse_config(doc))
    vel = case.fields["velocity"]
    fields = (FieldArray("velocity", POINT, 3, vel.ravel(), comp_stride=case.n_points),
              FieldArray("temperature", POINT, 1, case.fields["temperature"].ravel()))
    blk = SemBlock(case.n_elements, case.x, case.y, case.z, fields=fields)
    total = 0
    for step in range(5):
        reps = br.update(Snapshot(0.1 * step, step, 0, (blk,)))
        assert all(r.error is None for r in reps), reps
        total += sum(r.bytes_written for r in reps)
    names = sorted(p.name for p in (tmp_path / "out").glob("*.ppm"))
    assert names == [f"step{s:06d}_temperature.ppm" for s in (0, 2, 4)]
    assert total == 3 * (len("P6\n80 60\n255\n") + 80 * 60 * 3)
    # image content = oracle
    sink = br.sinks[0]
    cf = O.CaseFields(case.x, case.y, case.z, case.fields)
    surf = [("iso", "Q", 0.5), ("iso", "temperature", 0.6), ("slice", (0.3, 1.0, 0.2), 0.9)]
    rgba, _, _, _ = O.pipeline_mt(cf, surf, "temperature", sink.last.view, 80, 60, 4)
    raw = (tmp_path / "out" / "step000004_temperature.ppm").read_bytes()
    assert raw[len("P6\n80 60\n255\n"):] == rgba[..., :3].tobytes()
    sums = br.finalize()
    assert sums[0].invocations == 3 and sums[1].invocations == 5


def test_insitu_sink_async_write_same_files(tmp_path):
    """async_write=1 (PPM of step i written while step i+1 runs) leaves the
    same files, byte for byte, as the synchronous sink once finalize() ran."""
    from paper_2312_09888_b200.sinks import InsituSink

    case = synth.box(nel=(3, 2, 2))
    vel = case.fields["velocity"]

    def blk(st):      # a different temperature every step: a write racing the next step would show
        t = case.fields["temperature"].ravel() + 0.07 * st
        fields = (FieldArray("velocity", POINT, 3, vel.ravel(), comp_stride=case.n_points),
                  FieldArray("temperature", POINT, 1, t))
        return SemBlock(case.n_elements, case.x, case.y, case.z, fields=fields)

    out = {}
    for mode in ("0", "1"):
        d = tmp_path / f"w{mode}"
        sink = InsituSink({"dir": str(d), "iso": "Q=0.5;temperature=0.6", "field": "temperature",
                           "width": "96", "height": "64", "view": "30,40", "async_write": mode})
        assert sink.async_write == (mode == "1")
        n = sum(sink.consume(Snapshot(0.1 * st, st, 0, (blk(st),))) for st in range(4))
        sink.finalize()
        out[mode] = {p.name: p.read_bytes() for p in sorted(d.glob("*.ppm"))}
        assert n == 4 * (len("P6\n96 64\n255\n") + 96 * 64 * 3)
    assert list(out["0"]) == [f"step{s:06d}_temperature.ppm" for s in range(4)]
    assert out["0"] == out["1"]
    assert len(set(out["0"].values())) == 4


def test_failing_insitu_sink_is_isolated(tmp_path):
    doc = (f'<sensei><analysis type="insitu" frequency="1" dir="{tmp_path}/o" iso="nope=1" field="temperature"/>'
           f'<analysis type="null" frequency="1"/></sensei>')
    br = initialize(parse_config(doc))
    case = synth.box(nel=(1, 1, 1))
    blk = SemBlock(1, case.x, case.y, case.z,
                   fields=(FieldArray("temperature", POINT, 1, case.fields["temperature"].ravel()),))
    reps = br.update(Snapshot(0.0, 0, 0, (blk,)))
    assert "ValueError" in reps[0].error and reps[1].error is None


@pytest.mark.parametrize("wh", [(7, 5), (80, 60), (1, 1), (13, 3)])
def test_image_ppm_equals_write_ppm_bytes(tmp_path, wh):
    """GPU RGB pack + pinned PPM buffer == write_ppm(ImageRGB(rgba[..., :3]))
    byte for byte, including pixel counts that are not a multiple of 4."""
    from paper_2312_09888_b200.adaptor import SemDataAdaptor
    from paper_2312_09888_b200.analysis import InsituAnalysis, Pipeline, Surface
    from paper_2312_09888_b200.context import Context
    from paper_2312_09888_b200.sinks import ImageRGB, write_ppm

    w, h = wh
    case = synth.box(nel=(2, 2, 2))
    ctx = Context(0)
    da = SemDataAdaptor(ctx)
    fields = tuple(FieldArray(k, POINT, v.shape[0], v.ravel(), comp_stride=case.n_points)
                   for k, v in case.fields.items())
    da.initialize(Snapshot(0.0, 0, 0, (SemBlock(case.n_elements, case.x, case.y, case.z, fields=fields),)))
    res = InsituAnalysis(Pipeline(surfaces=(Surface("iso", "temperature", 0.6),), color_field="temperature",
                                  width=w, height=h)).execute(da)
    n = write_ppm(ImageRGB(w, h, res.rgba[..., :3].tobytes()), tmp_path / "a.ppm")
    ppm = bytes(ctx.image_ppm())
    assert len(ppm) == n and ppm == (tmp_path / "a.ppm").read_bytes()
    ctx.close()


def test_gpu_colormap_equals_np_interp_on_2m_samples(ctx):
    """SURVEY.md §8c pin: the GPU colormap (structured renderer, exact grid
    sampling with vmin=0, vmax=1 so t = value) against the reference's own
    formula -- np.interp per channel then floor(v + 0.5) (sinks.py:201-209)
    -- on 2,097,152 samples including the anchors, clipping and exact halves."""
    from paper_2312_09888_b200.device import DeviceArray

    ni, nj = 16384, 128
    rng = np.random.default_rng(123)
    t = rng.uniform(-0.2, 1.2, ni * nj)
    halves = (np.arange(0, 196) + 0.5 - 59) / 392.0
    special = np.array([0.0, 0.5, 1.0, -0.0, 0.25, 0.75, np.nextafter(0.5, 0), np.nextafter(0.5, 1), 1e-300])
    t[:special.size] = special
    t[special.size:special.size + halves.size] = halves
    grid = t.reshape(nj, ni)                         # row j = y index (x fastest)
    d = DeviceArray.empty(ctx, (t.size,), np.float64)
    d.upload(np.ascontiguousarray(grid).ravel())
    rgb = DeviceArray.empty(ctx, (ni * nj * 3,), np.uint8)
    ctx.render_structured([(d, ni)], nj, 1, 0, ni, nj, 0.0, 1.0, rgb)
    img = rgb.to_host().reshape(nj, ni, 3)[::-1]     # row 0 = top = largest y
    tc = np.clip(grid, 0.0, 1.0)
    exp = np.empty((nj, ni, 3), np.uint8)
    for ch, col in enumerate(((59, 255, 180), (76, 255, 4), (192, 255, 38))):
        exp[..., ch] = np.floor(np.interp(tc, [0.0, 0.5, 1.0], col) + 0.5).astype(np.uint8)
    assert np.array_equal(img, exp), int((img != exp).any(-1).sum())


def test_device_memory_flat_over_many_steps():
    """insitu + stats + checkpoint sinks for 60 steps: no per-step device
    allocations leak (tools/soak.py runs the long version)."""
    import subprocess
    import sys

    r = subprocess.run([sys.executable, "tools/soak.py", "60"], capture_output=True, text=True,
                       cwd=__import__("os").path.dirname(__import__("os").path.dirname(__file__)))
    assert r.returncode == 0 and "soak ok" in r.stdout, r.stdout + r.stderr
