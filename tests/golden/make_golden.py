"""Generate golden vectors from the REFERENCE implementation (run here, where
/root/reference exists; the outputs are committed, the GPU box never reads
/root/reference).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Fixtures (tests/golden/*.npz):
  colormap.npz   DEFAULT_COLORMAP.apply (reference sinks.py:201-213) on
                 seeded t samples incl. anchors, clipping, exact halves
  render.npz     reference `render` (sinks.py:245-295) on seeded snapshots:
                 scalar + ':mag', 1..4 blocks (assemble_global,
                 data_model.py:188-225), explicit ranges, degenerate range,
                 odd sizes, 1-pixel images, 3D (nk > 1) blocks
  ppm.npz        write_ppm byte streams (sinks.py:298-303)
  checkpoint.npz checkpoint_write files (sinks.py:60-102): binary and ascii,
                 point + cell fields, 1..3 blocks, title line round-trip values
"""
from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from nekmini.data_model import CELL, POINT, Block, FieldArray, Snapshot  # noqa: E402
from nekmini.sinks import DEFAULT_COLORMAP, ImageRGB, checkpoint_write, render, write_ppm  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from cases import CHECKPOINT_CASES, RENDER_CASES, checkpoint_arrays, colormap_samples, snapshot_arrays  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def snapshot(seed, ni, nj, nk=1, nblocks=1, comps=2):
    blocks = []
    for temp, vel, ext in snapshot_arrays(seed, ni, nj, nk, nblocks, comps):
        fields = (FieldArray("temperature", POINT, 1, temp), FieldArray("velocity", POINT, comps, vel))
        blocks.append(Block((ext[0] * 0.5, 0.0, 0.0), (0.5, 0.25, 1.0), ext, fields))
    return Snapshot(time=0.0, step=3, producer_id=0, blocks=tuple(blocks))


def main():
    t = colormap_samples()
    rgb = DEFAULT_COLORMAP.apply(t)
    np.savez_compressed(os.path.join(HERE, "colormap.npz"), rgb=rgb)

    images = {}
    for case in RENDER_CASES:
        seed, ni, nj, nk, nb, comps, field, w, h, vmin, vmax = case
        s = snapshot(seed, ni, nj, nk, nb, comps)
        img = render(s, field, DEFAULT_COLORMAP, w, h, vmin, vmax)
        images[f"case{seed}"] = np.frombuffer(img.pixels, np.uint8).copy()
    np.savez_compressed(os.path.join(HERE, "render.npz"), **images)

    with tempfile.TemporaryDirectory() as d:
        ppms = {}
        for (w, h) in ((1, 1), (3, 2), (256, 256)):
            rng = np.random.default_rng(w * 1000 + h)
            px = rng.integers(0, 256, size=3 * w * h, dtype=np.uint8).tobytes()
            p = os.path.join(d, "x.ppm")
            n = write_ppm(ImageRGB(w, h, px), p)
            raw = open(p, "rb").read()
            assert n == len(raw)
            ppms[f"ppm_{w}x{h}"] = np.frombuffer(raw, np.uint8).copy()
    np.savez_compressed(os.path.join(HERE, "ppm.npz"), **ppms)

    with tempfile.TemporaryDirectory() as d:
        files = {}
        for case in CHECKPOINT_CASES:
            seed, ni, nj, nk, nb, comps, cellf, fmt, step, prod, tm = case
            blocks = []
            for temp, vel, pres, ext in checkpoint_arrays(seed, ni, nj, nk, nb, comps, cellf):
                fields = [FieldArray("temperature", POINT, 1, temp), FieldArray("velocity", POINT, comps, vel)]
                if pres is not None:
                    fields.append(FieldArray("pressure", CELL, 1, pres))
                blocks.append(Block((ext[0] * 0.5, -1.25, 1e-3), (0.5, 0.25, 1.0 / 3.0), ext, tuple(fields)))
            paths, total = checkpoint_write(Snapshot(tm, step, prod, tuple(blocks)), d, fmt)
            assert total == sum(os.path.getsize(p) for p in paths)
            for bi, p in enumerate(paths):
                files[f"case{seed}_b{bi}"] = np.frombuffer(open(p, "rb").read(), np.uint8).copy()
                files[f"case{seed}_b{bi}_name"] = np.array(os.path.basename(p))
        np.savez_compressed(os.path.join(HERE, "checkpoint.npz"), **files)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
