"""Seeded inputs of the golden fixtures (pure numpy; no reference import, so
tests on the GPU box can rebuild the inputs while the expected outputs come
from the committed .npz files made by make_golden.py)."""
from __future__ import annotations

import numpy as np


def colormap_samples(seed: int = 20231215, n: int = 200_000) -> np.ndarray:
    rng = np.random.default_rng(seed)
    t = rng.uniform(-0.25, 1.25, size=n)
    special = np.array([0.0, 0.5, 1.0, -0.0, 0.25, 0.75, 1e-300, 0.5 - 1e-17, 0.5 + 1e-16,
                        1.0 - 1e-16, -3.0, 5.0, np.nextafter(0.5, 0), np.nextafter(0.5, 1)])
    # values whose red channel lands on k + 0.5 (the floor(v + 0.5) rounding rule)
    halves = (np.arange(0, 196) + 0.5 - 59) / 392.0
    halves = halves[(halves >= 0) & (halves < 0.5)]
    return np.concatenate([special, halves, t])


def snapshot_arrays(seed, ni, nj, nk=1, nblocks=1, comps=2):
    """Per block: (temperature[npts], velocity[comps*npts] AoS, extents)."""
    rng = np.random.default_rng(seed)
    out = []
    for b in range(nblocks):
        npts = ni * nj * nk
        temp = rng.standard_normal(npts)
        vel = rng.standard_normal(comps * npts)
        o = b * ni
        out.append((temp, vel, (o, o + ni - 1, 0, nj - 1, 0, nk - 1)))
    return out


RENDER_CASES = [
    # (seed, ni, nj, nk, nblocks, comps, field, w, h, vmin, vmax)
    (1, 7, 5, 1, 1, 2, "temperature", 11, 9, None, None),
    (2, 7, 5, 1, 1, 2, "velocity:mag", 11, 9, None, None),
    (3, 16, 12, 1, 4, 3, "velocity:mag", 64, 48, None, None),
    (4, 16, 12, 1, 3, 2, "temperature", 37, 23, -0.5, 0.75),
    (5, 5, 4, 3, 2, 3, "velocity:mag", 20, 30, None, None),
    (6, 2, 2, 1, 1, 2, "temperature", 1, 1, None, None),
    (7, 9, 1, 1, 1, 2, "temperature", 8, 8, None, None),
    (8, 1, 6, 1, 1, 2, "temperature", 4, 5, None, None),
    (9, 30, 20, 1, 2, 2, "temperature", 256, 256, None, None),
    (10, 6, 6, 1, 1, 2, "temperature", 13, 7, 2.0, 2.0),
]


def cell_count(ni, nj, nk):
    """Block.cell_count (reference data_model.py:83-86): a flat axis counts 1."""
    return max(ni - 1, 1) * max(nj - 1, 1) * max(nk - 1, 1)


CHECKPOINT_CASES = [
    # (seed, ni, nj, nk, nblocks, comps, with_cell_field, fmt, step, producer, time)
    (21, 6, 5, 1, 1, 2, False, "binary", 0, 0, 0.0),
    (22, 6, 5, 1, 1, 3, True, "binary", 17, 3, 0.1 + 0.2),
    (23, 4, 3, 2, 3, 2, True, "binary", 400, 1, 12.5),
    (24, 5, 4, 1, 2, 2, True, "ascii", 9, 2, 1.0 / 3.0),
    (25, 1, 1, 1, 1, 1, False, "ascii", 1, 0, -2.0),
]


def checkpoint_arrays(seed, ni, nj, nk, nblocks, comps, with_cell):
    """Per block: (temperature, velocity AoS, pressure cell field or None, extents)."""
    rng = np.random.default_rng(seed)
    out = []
    for b in range(nblocks):
        npts = ni * nj * nk
        temp = rng.standard_normal(npts) * 10.0 ** rng.integers(-5, 6, npts)
        vel = rng.standard_normal(comps * npts)
        pres = rng.standard_normal(cell_count(ni, nj, nk)) if with_cell else None
        o = b * ni
        out.append((temp, vel, pres, (o, o + ni - 1, 0, nj - 1, 0, nk - 1)))
    return out
