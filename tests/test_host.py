"""Host-side logic (no GPU): C-ABI surface, bridge semantics mirrored from the
reference's tests (reference pkg/tests/test_bridge.py), pipeline parsing,
camera, data model validation, synthetic meshes."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

from paper_2312_09888_b200 import _native as N
from paper_2312_09888_b200 import bridge as bridge_mod
from paper_2312_09888_b200 import synth
from paper_2312_09888_b200.analysis import Pipeline, Surface, ortho_view, pipeline_from_params
from paper_2312_09888_b200.bridge import (AnalysisSpec, Bridge, BridgeConfig, ConfigError, parse_config,
                                          should_trigger)
from paper_2312_09888_b200.data_model import (CELL, POINT, Block, FieldArray, SchemaMismatch, SemBlock,
                                              Snapshot, assemble_global, metadata_of, validate_snapshot)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# ------------------------------------------------------------------ C ABI


def _header_functions():
    with open(os.path.join(ROOT, "include", "nekb200.h")) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(nkb_[a-z_0-9]+)\s*\(", text)))


def test_library_loads_and_exports_every_header_symbol():
    lib = ctypes.CDLL(N.LIB_PATH)
    names = _header_functions()
    assert len(names) >= 30
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(N.EXPORTED), set(names) ^ set(N.EXPORTED)
    assert lib.nkb_abi_version() == 1


def test_status_codes_map_to_reference_exceptions():
    L = N.lib()
    x = np.zeros(3)
    rc = L.nkb_gll(0, x.ctypes.data, None)
    assert rc == N.NKB_EINVAL
    with pytest.raises(ValueError, match="order"):
        N.check(rc)
    assert b"order" in L.nkb_last_error()


def test_gll_through_abi_without_gpu():
    from paper_2312_09888_b200.context import gll

    x, D = gll(7)
    assert x[0] == -1.0 and x[-1] == 1.0 and D.shape == (8, 8)


def test_synth_gll_constants_match_library_and_oracle():
    # synth.py spells out the N=7 nodes so case generation maps no native
    # library (the bench's reference arm); they must be the library's bits
    from oracle import oracle as orc
    from paper_2312_09888_b200 import synth
    from paper_2312_09888_b200.context import gll

    x, _ = gll(7)
    xo, _ = orc.gll(7)
    assert np.array_equal(synth.GLL7.view(np.uint64), x.view(np.uint64))
    assert np.array_equal(synth.GLL7.view(np.uint64), xo.view(np.uint64))


def test_pipeline_struct_layout_matches_header():
    # offsets the C compiler assigns must match ctypes (checked via a tiny C program)
    import subprocess
    import tempfile

    src = r"""
    #include <stdio.h>
    #include <stddef.h>
    #include "nekb200.h"
    int main(){printf("%zu %zu %zu %zu %zu %zu %zu\n", sizeof(nkb_pipeline), offsetof(nkb_pipeline, view),
      offsetof(nkb_pipeline, anchor_rgb), offsetof(nkb_pipeline, timing), sizeof(nkb_report),
      sizeof(nkb_mesh_metadata), offsetof(nkb_report, reran)); return 0;}
    """
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        open(c, "w").write(src)
        exe = os.path.join(d, "t")
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe], check=True)
        got = [int(v) for v in subprocess.run([exe], capture_output=True, text=True).stdout.split()]
    P = N.NkbPipeline
    assert got == [ctypes.sizeof(P), P.view.offset, P.anchor_rgb.offset, P.timing.offset,
                   ctypes.sizeof(N.NkbReport), ctypes.sizeof(N.NkbMeshMetadata), N.NkbReport.reran.offset]


# ----------------------------------------------------- bridge (reference semantics)

CATALYST_DOC = """<sensei>
  <analysis type="catalyst" pipeline="pythonscript" filename="analysis.py" frequency="100" />
</sensei>
"""


def test_catalyst_document_parses_verbatim():
    cfg = parse_config(CATALYST_DOC)
    assert len(cfg.specs) == 1 and cfg.specs[0].kind == "render" and cfg.specs[0].frequency == 100


def test_insitu_kind_and_attributes():
    cfg = parse_config('<sensei><analysis type="insitu" frequency="10" iso="Q=0.1" slice="y=0" '
                       'field="temperature" width="64" height="32" bogus="1"/></sensei>')
    s = cfg.specs[0]
    assert s.kind == "insitu" and s.frequency == 10 and "bogus" not in s.params
    p = pipeline_from_params(s.params)
    assert p.width == 64 and p.height == 32 and p.color_field == "temperature"
    assert p.surfaces == (Surface("iso", "Q", 0.1), Surface("slice", value=0.0, normal=(0.0, 1.0, 0.0)))


@pytest.mark.parametrize("doc,match", [
    ('<sensei><analysis type="frobnicate" frequency="1"/></sensei>', "unknown analysis kind"),
    ('<sensei><analysis type="null" frequency="0"/></sensei>', "frequency"),
    ('<sensei><analysis type="null" frequency="x"/></sensei>', "integer"),
    ("<sensei><analysis", "malformed"),
    ("<other/>", "root element"),
    ('<sensei><analysis frequency="1"/></sensei>', "missing 'type'"),
    ('<sensei><analysis type="stats" frequency="1"/></sensei>', "requires a 'path'"),
])
def test_config_errors(doc, match):
    with pytest.raises(ConfigError, match=match):
        parse_config(doc)


def test_empty_document_and_unknown_element(caplog):
    assert parse_config("<sensei></sensei>").specs == ()
    with caplog.at_level("WARNING"):
        cfg = parse_config('<sensei><foo/><analysis type="null" frequency="2" zap="1"/></sensei>')
    assert cfg.specs[0].kind == "null"
    msgs = " ".join(r.message for r in caplog.records)
    assert "zap" in msgs and "foo" in msgs


@pytest.mark.parametrize("freq,step_no,at_zero,expected", [
    (100, 100, True, True), (100, 101, True, False), (100, 0, False, False), (100, 0, True, True),
    (1, 7, False, True)])
def test_should_trigger(freq, step_no, at_zero, expected):
    assert should_trigger(AnalysisSpec("null", freq), step_no, at_zero) is expected


def test_should_trigger_negative_step():
    with pytest.raises(ValueError):
        should_trigger(AnalysisSpec("null", 1), -1)


def _struct_snapshot(step=0):
    f = FieldArray("temperature", POINT, 1, np.arange(16.0))
    return Snapshot(0.0, step, 0, (Block((0, 0, 0), (1, 1, 1), (0, 3, 0, 3, 0, 0), (f,)),))


def test_trigger_count_over_run():
    br = Bridge(BridgeConfig((AnalysisSpec("null", 100),), trigger_at_step_zero=False))
    n = sum(len(br.update(_struct_snapshot(s))) for s in range(1, 3001))
    assert n == 30 and br.finalize()[0].invocations == 30


def test_non_monotone_and_invalid_snapshot():
    br = Bridge(BridgeConfig((AnalysisSpec("null", 1),)))
    br.update(_struct_snapshot(5))
    with pytest.raises(ValueError, match="non-increasing"):
        br.update(_struct_snapshot(5))
    with pytest.raises(ValueError, match="invalid snapshot"):
        br.update(Snapshot(0.0, 9, 0, ()))


class _Boom:
    def consume(self, s):
        raise IOError("disk on fire")

    def finalize(self):
        raise RuntimeError("flush failed")


def test_sink_failure_isolated_and_counted():
    br = Bridge(BridgeConfig((AnalysisSpec("null", 1), AnalysisSpec("null", 1))))
    br.sinks[0] = _Boom()
    reps = br.update(_struct_snapshot(0))
    assert "disk on fire" in reps[0].error and reps[1].error is None
    sums = br.finalize()
    assert sums[0].failures == 2 and sums[1].invocations == 1   # consume + finalize failures


def test_unwritable_output_fails_at_initialize(tmp_path):
    blocker = tmp_path / "blocker"
    blocker.write_text("")
    doc = f'<sensei><analysis type="render" frequency="1" dir="{blocker}/img"/></sensei>'
    with pytest.raises(OSError):
        bridge_mod.initialize(parse_config(doc))


# ------------------------------------------------------------- pipeline / camera


def test_ortho_view_maps_bounds_into_image():
    b = (0.0, 2.0, 0.0, 1.0, 0.0, 1.0)
    for az, el in ((0, 90), (35, 30), (-60, 25), (90, 0)):
        V = np.array(ortho_view(b, 200, 100, az, el)).reshape(3, 4)
        corners = np.array([[x, y, z, 1.0] for x in b[:2] for y in b[2:4] for z in b[4:]])
        s = corners @ V.T
        assert s[:, 0].min() >= 0 and s[:, 0].max() <= 200
        assert s[:, 1].min() >= 0 and s[:, 1].max() <= 100
        assert s[:, 2].min() > 0 and s[:, 2].max() < 1


def test_ortho_view_top_down_orientation():
    V = np.array(ortho_view((0, 1, 0, 1, 0, 1), 100, 100, 0, 90)).reshape(3, 4)
    hi_y = V @ [0.5, 1.0, 0.5, 1]
    lo_y = V @ [0.5, 0.0, 0.5, 1]
    assert hi_y[1] < lo_y[1]            # +y is up: smaller row (row 0 = top)
    near = V @ [0.5, 0.5, 1.0, 1]
    far = V @ [0.5, 0.5, 0.0, 1]
    assert near[2] < far[2]             # camera above +z: larger z is nearer


def test_pipeline_native_roundtrip():
    p = Pipeline(surfaces=(Surface("iso", "Q", 0.25), Surface("slice", value=1.0, normal=(0, 0, 1))),
                 color_field="temperature", width=33, height=17, vmin=0.0)
    n = p.native(tuple(range(12)))
    assert n.n_surfaces == 2 and n.surfaces[0].field == b"Q" and n.surfaces[1].kind == N.NKB_SURF_SLICE
    assert n.width == 33 and n.vmin == 0.0 and math.isnan(n.vmax) and n.n_anchors == 0
    with pytest.raises(ValueError):
        Pipeline(surfaces=(Surface("blob"),)).native(tuple(range(12)))


def test_pipeline_params_errors():
    with pytest.raises(ValueError):
        pipeline_from_params({"iso": "Q"})
    with pytest.raises(ValueError):
        pipeline_from_params({"slice": "w=1"})


# --------------------------------------------------------------- data model


def test_structured_validation_matches_reference_rules():
    good = _struct_snapshot()
    assert validate_snapshot(good) == []
    bad = Snapshot(0.0, -1, 0, (Block((0, 0, 0), (1, 0, 1), (0, 3, 0, 3, 0, 0),
                                      (FieldArray("t", POINT, 1, np.zeros(5)),)),))
    v = validate_snapshot(bad)
    assert "negative step" in v and any("spacing" in m for m in v) and any("length" in m for m in v)


def test_assemble_global_index_arithmetic():
    # reference tests/test_data_model.py:74-89: i=5,j=3 <-> tile 2 (1,3)
    blocks = []
    for b in range(3):
        vals = np.arange(2 * 4, dtype=float) + 100 * b
        f = FieldArray("t", POINT, 1, vals)
        blocks.append(Block((0, 0, 0), (1, 1, 1), (2 * b, 2 * b + 1, 0, 3, 0, 0), (f,)))
    g = assemble_global(blocks)
    grid = g.field_named("t").values.reshape(4, 6)
    assert grid[3, 5] == 200 + 1 + 2 * 3
    assert g.extents == (0, 5, 0, 3, 0, 0)
    with pytest.raises(SchemaMismatch):
        assemble_global([blocks[0], Block((0, 0, 0), (2, 1, 1), (2, 3, 0, 3, 0, 0), blocks[1].fields)])


def test_sem_block_validation_and_metadata():
    c = synth.box(nel=(2, 1, 1))
    vel = c.fields["velocity"]
    blk = SemBlock(c.n_elements, c.x, c.y, c.z,
                   fields=(FieldArray("velocity", POINT, 3, vel.ravel(), comp_stride=c.n_points),))
    s = Snapshot(0.0, 0, 0, (blk,))
    assert validate_snapshot(s) == []
    m = metadata_of(s)
    assert (m.n_elements, m.n_points, m.n_cells, m.cell_type) == (2, 1024, 686, 12)
    short = SemBlock(2, c.x[:100], c.y, c.z)
    assert any("coordinate x" in v for v in validate_snapshot(Snapshot(0.0, 0, 0, (short,))))


# ------------------------------------------------------------ synthetic meshes


def test_partition_covers_all_elements():
    E = 1000
    parts = [synth.partition(E, r, 7) for r in range(7)]
    assert parts[0][0] == 0 and parts[-1][1] == E
    assert all(parts[i][1] == parts[i + 1][0] for i in range(6))


def test_partitioned_case_equals_slice_of_full():
    full = synth.box(nel=(3, 2, 2))
    part = synth.box(5, 9, nel=(3, 2, 2))
    sl = slice(5 * 512, 9 * 512)
    assert np.array_equal(part.x, full.x[sl]) and np.array_equal(part.fields["velocity"],
                                                                 full.fields["velocity"][:, sl])


def test_cylinder_mesh_is_curved_and_inside_unit_disk():
    c = synth.rbc_cylinder(0, 64, nel=(4, 4, 4))
    r = np.hypot(c.x, c.y)
    assert r.max() <= 1.0 + 1e-12
    assert c.fields["temperature"].shape == (1, 64 * 512)


def test_kinds_of_the_reference_and_the_sem_path():
    """Every reference sink kind exists (render, stats, checkpoint, null;
    reference sinks.py:405-410) plus insitu / transit; attributes are
    filtered per kind like the reference's _KNOWN_ATTRS (bridge.py:34-39)."""
    from paper_2312_09888_b200.bridge import KINDS
    from paper_2312_09888_b200.sinks import _SINK_TYPES

    for k in ("render", "stats", "checkpoint", "null", "insitu", "transit"):
        assert k in KINDS and k in _SINK_TYPES
    cfg = parse_config('<sensei><analysis type="stats" path="/tmp/x.csv" frequency="3" dir="d"/>'
                       '<analysis type="checkpoint" dir="ck" format="ascii" arrays="Q" width="5"/>'
                       '<analysis type="transit" endpoint="1" iso="Q=1" continuous="1"/></sensei>')
    st, ck, tr = cfg.specs
    assert st.params == {"path": "/tmp/x.csv"} and st.frequency == 3
    assert ck.params == {"dir": "ck", "format": "ascii", "arrays": "Q"}
    assert tr.params == {"endpoint": "1", "iso": "Q=1"}          # continuous is an insitu-only attribute


def test_stats_and_checkpoint_sinks_construct_without_gpu(tmp_path):
    """Constructing sinks needs no GPU (only consume does), and output
    locations are probed like the reference's (_probe_writable)."""
    from paper_2312_09888_b200.sinks import CheckpointSink, StatsSink

    StatsSink({"path": str(tmp_path / "a" / "s.csv")})
    assert (tmp_path / "a" / "s.csv").read_text() == "step,time,field,min,max,mean\n"
    CheckpointSink({"dir": str(tmp_path / "ck")})
    with pytest.raises(ValueError, match="ascii or binary"):
        CheckpointSink({"dir": str(tmp_path / "ck"), "format": "hdf5"})


def test_perspective_view_maps_sphere_into_image():
    """The pinhole camera puts the bounds' centre at the image centre with a
    depth in (0, 1), the nearest / farthest points of the bounding sphere at
    depth ~0 / ~1, and keeps +z up for an elevation of 0."""
    import math

    from paper_2312_09888_b200.analysis import perspective_view

    b = (0.0, 2.0, -1.0, 1.0, 0.0, 1.0)
    v = np.array(perspective_view(b, 200, 100, azimuth=30.0, elevation=0.0, fov=40.0, margin=1.0))
    V, P = v[:12].reshape(3, 4), v[12:]

    def proj(x):
        h = np.append(x, 1.0)
        return V @ h / (P @ h)

    c = np.array([1.0, 0.0, 0.5])
    sx, sy, sz = proj(c)
    assert abs(sx - 100) < 1e-9 and abs(sy - 50) < 1e-9 and 0 < sz < 1
    r = 0.5 * math.sqrt(4 + 4 + 1)
    d = np.array([math.cos(math.radians(30)), math.sin(math.radians(30)), 0.0])
    assert abs(proj(c + r * d)[2]) < 1e-12 and abs(proj(c - r * d)[2] - 1.0) < 1e-12
    assert proj(c + [0, 0, 0.4])[1] < sy                       # higher z -> smaller row (up)


def test_insitu_async_write_attribute_parses_and_reaches_the_sink(tmp_path):
    """async_write is an insitu attribute: the bridge keeps
    it and the sink built from the parsed params writes on a writer thread."""
    from paper_2312_09888_b200.sinks import InsituSink

    cfg = parse_config(f'<sensei><analysis type="insitu" frequency="1" iso="Q=1" async_write="1" '
                       f'dir="{tmp_path}"/></sensei>')
    s = cfg.specs[0]
    assert s.params["async_write"] == "1"
    assert InsituSink(s.params).async_write


def test_insitu_sink_without_composite_writes_one_file_per_rank(tmp_path):
    """composite="0" on several ranks: each rank writes its own partial image
    under a rank-suffixed name (no clobbering), and probes the directory."""
    from paper_2312_09888_b200.sinks import InsituSink

    class _Comm:
        def __init__(self, rank, size):
            self.rank, self.size = rank, size

    d = tmp_path / "parts"
    s1 = InsituSink({"dir": str(d), "composite": "0", "iso": "Q=1"}, comm=_Comm(1, 2))
    assert s1.per_rank and d.is_dir()
    s0 = InsituSink({"dir": str(tmp_path / "one"), "iso": "Q=1"}, comm=_Comm(1, 2))
    assert not s0.per_rank and not (tmp_path / "one").exists()      # composite: rank 0 writes


def test_bench_balanced_cuts():
    """bench.py --partition work: contiguous ranges of equal surface-pass cost."""
    import importlib.util
    import os

    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(os.path.dirname(__file__), "..", "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    # uniform work: the equal partition
    assert bench.balanced_cuts(np.zeros(100, np.int64), 4) == [0, 25, 50, 75, 100]
    # all triangles at the end: the last rank gets few elements
    t = np.zeros(1000, np.int64)
    t[900:] = 1000
    cuts = bench.balanced_cuts(t, 4, weight=0.1)
    cost = 1.0 + 0.1 * t
    parts = [cost[cuts[k]:cuts[k + 1]].sum() for k in range(4)]
    assert cuts[0] == 0 and cuts[-1] == 1000 and all(b > a for a, b in zip(cuts, cuts[1:]))
    assert max(parts) / min(parts) < 1.05
    # more ranks than heavy elements, and the degenerate tiny case: ranges stay non-empty
    cuts = bench.balanced_cuts(np.array([0, 0, 10**6, 0, 0]), 4)
    assert all(b > a for a, b in zip(cuts, cuts[1:])) and cuts[-1] == 5
    assert bench.balanced_cuts(np.zeros(4, np.int64), 4) == [0, 1, 2, 3, 4]
