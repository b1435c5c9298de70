"""Checkpoint files.  Structured snapshots: byte-identical to the reference's
checkpoint_write (golden files from tests/golden/make_golden.py) and read
back bit-exactly.  SEM partitions (GPU-encoded UNSTRUCTURED_GRID): see the
gpu test below -- points, connectivity, types and arrays round-trip against
the host arrays and the oracle."""
import os

import numpy as np
import pytest
from cases import CHECKPOINT_CASES, checkpoint_arrays

from paper_2312_09888_b200.data_model import CELL, POINT, Block, FieldArray, SemBlock, Snapshot
from paper_2312_09888_b200.vtk import CheckpointFormatError, checkpoint_read, checkpoint_write

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "checkpoint.npz"))


def _snapshot(case):
    seed, ni, nj, nk, nb, comps, cellf, fmt, step, prod, tm = case
    blocks = []
    for temp, vel, pres, ext in checkpoint_arrays(seed, ni, nj, nk, nb, comps, cellf):
        fields = [FieldArray("temperature", POINT, 1, temp), FieldArray("velocity", POINT, comps, vel)]
        if pres is not None:
            fields.append(FieldArray("pressure", CELL, 1, pres))
        blocks.append(Block((ext[0] * 0.5, -1.25, 1e-3), (0.5, 0.25, 1.0 / 3.0), ext, tuple(fields)))
    return Snapshot(tm, step, prod, tuple(blocks)), fmt


@pytest.mark.parametrize("case", CHECKPOINT_CASES, ids=[f"case{c[0]}" for c in CHECKPOINT_CASES])
def test_structured_checkpoint_bytes_match_reference(tmp_path, case):
    s, fmt = _snapshot(case)
    paths, total = checkpoint_write(s, tmp_path, fmt)
    assert total == sum(p.stat().st_size for p in paths)
    for bi, p in enumerate(paths):
        key = f"case{case[0]}_b{bi}"
        assert p.name == str(GOLD[key + "_name"])
        assert p.read_bytes() == GOLD[key].tobytes()


@pytest.mark.parametrize("case", CHECKPOINT_CASES, ids=[f"case{c[0]}" for c in CHECKPOINT_CASES])
def test_structured_checkpoint_round_trip(tmp_path, case):
    s, fmt = _snapshot(case)
    paths, _ = checkpoint_write(s, tmp_path, fmt)
    for bi, p in enumerate(paths):
        r = checkpoint_read(p)
        b = s.blocks[bi]
        assert (r.step, r.time) == (s.step, s.time)
        rb = r.blocks[0]
        assert rb.extents == b.extents and rb.origin == b.origin and rb.spacing == b.spacing
        for f in b.fields:
            g = rb.field_named(f.name)
            assert (g.association, g.components) == (f.association, f.components)
            assert np.array_equal(np.asarray(g.values).view(np.uint64), np.asarray(f.values).view(np.uint64))


def test_truncated_and_foreign_files(tmp_path):
    s, _ = _snapshot(CHECKPOINT_CASES[1])
    (p,), _ = checkpoint_write(s, tmp_path, "binary")
    raw = p.read_bytes()
    (tmp_path / "t.vtk").write_bytes(raw[:-50])
    with pytest.raises(CheckpointFormatError, match="truncated"):
        checkpoint_read(tmp_path / "t.vtk")
    (tmp_path / "f.vtk").write_bytes(b"hello\n")
    with pytest.raises(CheckpointFormatError, match="legacy VTK"):
        checkpoint_read(tmp_path / "f.vtk")
    with pytest.raises(ValueError, match="format"):
        checkpoint_write(s, tmp_path, "hdf5")


@pytest.mark.gpu
def test_sem_checkpoint_round_trip(tmp_path):
    """GPU-encoded UNSTRUCTURED_GRID of a SEM partition: every section reads
    back bit-exactly (points, VTK_HEXAHEDRON connectivity, types, the
    snapshot's fields in AoS order, and Q/|w| equal to the oracle)."""
    from oracle import oracle as O
    from paper_2312_09888_b200 import synth
    from paper_2312_09888_b200.bridge import initialize, parse_config
    from paper_2312_09888_b200.vtk import read_sem_vtk

    case = synth.box(nel=(3, 2, 2))
    vel = case.fields["velocity"]
    fields = (FieldArray("velocity", POINT, 3, vel.T.ravel()),
              FieldArray("temperature", POINT, 1, case.fields["temperature"].ravel()))
    blk = SemBlock(case.n_elements, case.x, case.y, case.z, fields=fields)
    doc = (f'<sensei><analysis type="checkpoint" dir="{tmp_path}/ck" arrays="Q,vorticity:mag" '
           f'frequency="1"/></sensei>')
    br = initialize(parse_config(doc))
    reps = br.update(Snapshot(0.75, 4, 2, (blk,)))
    assert reps[0].error is None, reps
    path = tmp_path / "ck" / "step000004_blk002.vtk"
    assert reps[0].bytes_written == path.stat().st_size
    r = read_sem_vtk(path)
    assert (r["step"], r["producer"], r["time"], r["n_elements"], r["order"]) == (4, 2, 0.75, 12, 7)
    assert np.array_equal(r["points"], np.stack([case.x, case.y, case.z], axis=1))
    e, a, b, c = np.meshgrid(np.arange(12), np.arange(7), np.arange(7), np.arange(7), indexing="ij")
    e, a, b, c = (v.transpose(0, 3, 2, 1).ravel() for v in (e, a, b, c))
    n0 = e * 512 + a + 8 * b + 64 * c
    assert np.array_equal(r["cells"], np.stack([n0, n0 + 1, n0 + 9, n0 + 8, n0 + 64, n0 + 65, n0 + 73, n0 + 72], 1))
    assert (r["types"] == 12).all()
    assert np.array_equal(r["arrays"]["velocity"], vel.T)
    assert np.array_equal(r["arrays"]["temperature"], case.fields["temperature"].ravel())
    q, wm, _, _ = O.derived(O.CaseFields(case.x, case.y, case.z, case.fields))
    assert np.array_equal(r["arrays"]["Q"], q) and np.array_equal(r["arrays"]["vorticity:mag"], wm)
