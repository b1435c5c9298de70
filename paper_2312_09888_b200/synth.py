"""Deterministic synthetic spectral-element meshes and fields (NekRS layout).

The reference's data source is its own 2D solver (solver.py, out of scope);
the north-star configurations (BASELINE.json `configs`) are NekRS cases whose
meshes are not available, so they are generated here, seeded with
`np.random.default_rng(seed)` as the reference seeds its solver
(solver.py:127).  Elements are ordered lexicographically (x fastest); inside
an element the GLL nodes are i-fastest: value(e,i,j,k) at e*512 + i + 8j + 64k.

Every generator takes an element range [e0, e1) so a rank builds only its
own contiguous partition (the NekRS-style split).

Configs:
  c1  Taylor-Green box [0,2pi]^3, 8^3 affine elements; Q iso 0.1, colour |u|
  c2  RBC cylinder, 32^3 curved elements (square->disk map); T iso 0.5,
      Q iso, slice y=0, colour T
  c3  turbPipe, 625 (25x25 disk) x 400 axial elements; Q iso, colour |w|
  c4  pebble bed, 128^3 box elements, dipoles around 146 spheres; slice
      z=0.5 + |u| iso, colour |u|
  c5  weak-scaling boxes of E = 65,536 .. 2,097,152 elements
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

NP = 8
NN = NP * NP * NP

# GLL nodes of order N=7, bit for bit what nkb_gll(7) (csrc/gll.cpp) and the
# oracle's orc_gll compute (tests/test_host.py checks all three agree).  They
# are spelled out here so that generating a synthetic case maps no native
# library: the bench's CPU reference arm builds the very same input bytes
# without loading libnekb200.
GLL7 = np.array([float.fromhex(h) for h in (
    "-0x1.0000000000000p+0", "-0x1.be54b988eafaap-1", "-0x1.2ef3538095d15p-1", "-0x1.aca5117fc1960p-3",
    "0x1.aca5117fc1960p-3", "0x1.2ef3538095d15p-1", "0x1.be54b988eafaap-1", "0x1.0000000000000p+0")])


@dataclass
class SemCase:
    name: str
    n_elements: int               # local
    e0: int                       # first global element of this partition
    n_elements_global: int
    x: np.ndarray
    y: np.ndarray
    z: np.ndarray
    fields: dict[str, np.ndarray] = field(default_factory=dict)   # name -> (ncomp, npts) SoA
    params: dict[str, str] = field(default_factory=dict)           # insitu sink attributes
    nel: tuple[int, int, int] | None = None                        # element lattice (global ids)

    @property
    def n_points(self) -> int:
        return self.n_elements * NN

    def global_ids(self) -> np.ndarray:
        """NekRS-style global node ids of this partition (int64, one per GLL copy)."""
        if self.nel is None:
            raise ValueError("this case has no element lattice")
        return lattice_ids(self.nel, self.e0, self.e0 + self.n_elements)


def _ref_coords(nel: tuple[int, int, int], e0: int, e1: int):
    """Logical coordinates in [0,1]^3 of every node of elements [e0, e1)."""
    t = (GLL7 + 1.0) / 2.0                         # GLL nodes on [0, 1]
    nx, ny, nz = nel
    e = np.arange(e0, e1)
    ex, ey, ez = e % nx, (e // nx) % ny, e // (nx * ny)
    # shape (E, k, j, i)
    X = (ex[:, None, None, None] + t[None, None, None, :]) / nx
    Y = (ey[:, None, None, None] + t[None, None, :, None]) / ny
    Z = (ez[:, None, None, None] + t[None, :, None, None]) / nz
    shp = (e1 - e0, NP, NP, NP)
    return (np.broadcast_to(X, shp).reshape(-1).copy(), np.broadcast_to(Y, shp).reshape(-1).copy(),
            np.broadcast_to(Z, shp).reshape(-1).copy())


def lattice_ids(nel: tuple[int, int, int], e0: int, e1: int) -> np.ndarray:
    """Global node ids on the (7 nx + 1) x (7 ny + 1) x (7 nz + 1) lattice of a
    structured element grid: copies of a node on shared faces, edges and
    corners get the same id."""
    nx, ny, nz = nel
    e = np.arange(e0, e1)
    ex, ey, ez = e % nx, (e // nx) % ny, e // (nx * ny)
    i = np.arange(NP)
    gx = (7 * ex)[:, None, None, None] + i[None, None, None, :]
    gy = (7 * ey)[:, None, None, None] + i[None, None, :, None]
    gz = (7 * ez)[:, None, None, None] + i[None, :, None, None]
    lx, ly = 7 * nx + 1, 7 * ny + 1
    return (gx + lx * (gy + ly * gz)).astype(np.int64).reshape(-1)


def partition(n_global: int, rank: int, nranks: int) -> tuple[int, int]:
    """Contiguous element range of `rank` (NekRS-style partition)."""
    return n_global * rank // nranks, n_global * (rank + 1) // nranks


def square_to_disk(u: np.ndarray, v: np.ndarray):
    """Elliptical grid map of [-1,1]^2 onto the unit disk (smooth, curved elements)."""
    return u * np.sqrt(1.0 - 0.5 * v * v), v * np.sqrt(1.0 - 0.5 * u * u)


def taylor_green(e0: int = 0, e1: int | None = None, n: int = 8) -> SemCase:
    E = n ** 3
    e1 = E if e1 is None else e1
    X, Y, Z = _ref_coords((n, n, n), e0, e1)
    L = 2.0 * math.pi
    x, y, z = L * X, L * Y, L * Z
    u = np.sin(x) * np.cos(y) * np.cos(z)
    v = -np.cos(x) * np.sin(y) * np.cos(z)
    w = np.zeros_like(x)
    p = (np.cos(2 * x) + np.cos(2 * y)) * (np.cos(2 * z) + 2.0) / 16.0
    return SemCase("c1", e1 - e0, e0, E, x, y, z,
                   {"velocity": np.stack([u, v, w]), "pressure": p[None]},
                   dict(PARAMS["c1"]), nel=(n, n, n))


def rbc_cylinder(e0: int = 0, e1: int | None = None, nel: tuple[int, int, int] = (32, 32, 32),
                 seed: int = 1) -> SemCase:
    """C2: Rayleigh-Benard cylinder (radius 1, height 1), curved elements."""
    E = nel[0] * nel[1] * nel[2]
    e1 = E if e1 is None else e1
    X, Y, Z = _ref_coords(nel, e0, e1)
    x, y = square_to_disk(2.0 * X - 1.0, 2.0 * Y - 1.0)
    z = Z
    rng = np.random.default_rng(seed)
    r = np.hypot(x, y)
    th = np.arctan2(y, x)
    T = 1.0 - z
    for _ in range(8):
        a, m, nz_, ph = rng.uniform(0.5, 1.0), int(rng.integers(0, 5)), int(rng.integers(1, 4)), rng.uniform(0, 2 * math.pi)
        T = T + 0.05 * a * r ** m * np.cos(m * th + ph) * np.sin(math.pi * nz_ * z)
    vel = []
    for c in range(3):
        acc = np.zeros_like(x)
        for _ in range(6):
            kx, ky, kz = rng.uniform(-4, 4, size=3)
            amp, ph = rng.uniform(0.1, 0.3), rng.uniform(0, 2 * math.pi)
            acc = acc + amp * np.sin(kx * x + ky * y + kz * z + ph)
        vel.append(acc)
    return SemCase("c2", e1 - e0, e0, E, x, y, z,
                   {"velocity": np.stack(vel), "temperature": T[None]},
                   dict(PARAMS["c2"]), nel=tuple(nel))


def turb_pipe(e0: int = 0, e1: int | None = None, nel: tuple[int, int, int] = (25, 25, 400),
              length: float = 20.0, seed: int = 2) -> SemCase:
    """C3: turbulent pipe, Poiseuille + 32 seeded Fourier modes (amplitude 0.1)."""
    E = nel[0] * nel[1] * nel[2]
    e1 = E if e1 is None else e1
    X, Y, Z = _ref_coords(nel, e0, e1)
    x, y = square_to_disk(2.0 * X - 1.0, 2.0 * Y - 1.0)
    z = length * Z
    rng = np.random.default_rng(seed)
    r2 = x * x + y * y
    vel = [np.zeros_like(x), np.zeros_like(x), 2.0 * (1.0 - r2)]
    for _ in range(32):
        k = rng.uniform(-6, 6, size=3)
        amp = 0.1 * rng.uniform(0.5, 1.0, size=3)
        ph = rng.uniform(0, 2 * math.pi, size=3)
        arg = k[0] * x + k[1] * y + k[2] * z
        damp = 1.0 - r2
        for c in range(3):
            vel[c] = vel[c] + amp[c] * damp * np.sin(arg + ph[c])
    return SemCase("c3", e1 - e0, e0, E, x, y, z, {"velocity": np.stack(vel)},
                   dict(PARAMS["c3"]), nel=tuple(nel))


def pebble_bed(e0: int = 0, e1: int | None = None, n: int = 128, n_spheres: int = 146, seed: int = 3) -> SemCase:
    """C4: unit box, uniform flow + potential-flow dipoles around seeded spheres."""
    E = n ** 3
    e1 = E if e1 is None else e1
    x, y, z = _ref_coords((n, n, n), e0, e1)
    rng = np.random.default_rng(seed)
    cs = rng.uniform(0.1, 0.9, size=(n_spheres, 3))
    rad = rng.uniform(0.03, 0.06, size=n_spheres)
    u = np.ones_like(x)
    v = np.zeros_like(x)
    w = np.zeros_like(x)
    for c, a in zip(cs, rad):
        dx, dy, dz = x - c[0], y - c[1], z - c[2]
        d2 = dx * dx + dy * dy + dz * dz + 1e-4
        d5 = d2 * d2 * np.sqrt(d2)
        k = 0.5 * a ** 3
        # dipole aligned with the mean flow (x): grad of k*dx/d^3
        u = u + k * (d2 - 3.0 * dx * dx) / d5
        v = v - k * 3.0 * dx * dy / d5
        w = w - k * 3.0 * dx * dz / d5
    return SemCase("c4", e1 - e0, e0, E, x, y, z, {"velocity": np.stack([u, v, w])},
                   dict(PARAMS["c4"]), nel=(n, n, n))


def box(e0: int = 0, e1: int | None = None, nel: tuple[int, int, int] = (4, 4, 4), seed: int = 0) -> SemCase:
    """Small smooth random box (parity tests / C5-style sweeps)."""
    E = nel[0] * nel[1] * nel[2]
    e1 = E if e1 is None else e1
    X, Y, Z = _ref_coords(nel, e0, e1)
    x, y, z = 2.0 * X, 1.5 * Y, 1.0 * Z
    rng = np.random.default_rng(seed)
    vel = []
    for c in range(3):
        acc = np.zeros_like(x)
        for _ in range(4):
            kx, ky, kz = rng.uniform(-3, 3, size=3)
            acc = acc + rng.uniform(0.2, 0.5) * np.sin(kx * x + ky * y + kz * z + rng.uniform(0, 6.28))
        vel.append(acc)
    T = np.cos(1.3 * x + 0.4) * np.sin(2.1 * y - 0.3) + z
    return SemCase("box", e1 - e0, e0, E, x, y, z, {"velocity": np.stack(vel), "temperature": T[None]},
                   {"iso": "Q=0.5;temperature=0.6", "slice": "0.3,1,0.2,0.9", "field": "temperature",
                    "view": "30,40"}, nel=tuple(nel))


def c5_lattice(n_elements: int) -> tuple[int, int, int]:
    """Element lattice of a C5 box: the most cubic (nx >= ny >= nz) power-of-two
    split, e.g. 65,536 = 64 x 32 x 32, 2,097,152 = 128 x 128 x 128."""
    if n_elements < 1 or n_elements & (n_elements - 1):
        raise ValueError(f"C5 element counts are powers of two, got {n_elements}")
    b = n_elements.bit_length() - 1
    ex = [b // 3 + (1 if i < b % 3 else 0) for i in range(3)]
    return (1 << ex[0], 1 << ex[1], 1 << ex[2])


C5_ELEMENTS = (65536, 131072, 262144, 524288, 1048576, 2097152)


def c5_box(e0: int = 0, e1: int | None = None, n_elements: int = 65536) -> SemCase:
    """C5: weak-scaling box (BASELINE configs[4]).  Cubic affine elements of
    edge pi/8 on the lattice `c5_lattice(E)`, periodic Taylor-Green velocity
    (the C1 flow, its period spanning 16 elements); full pipeline: Q iso,
    colour |u|."""
    nel = c5_lattice(n_elements)
    e1 = n_elements if e1 is None else e1
    X, Y, Z = _ref_coords(nel, e0, e1)
    h = math.pi / 8.0
    x, y, z = (h * nel[0]) * X, (h * nel[1]) * Y, (h * nel[2]) * Z
    u = np.sin(x) * np.cos(y) * np.cos(z)
    v = -np.cos(x) * np.sin(y) * np.cos(z)
    w = np.zeros_like(x)
    return SemCase("c5", e1 - e0, e0, n_elements, x, y, z, {"velocity": np.stack([u, v, w])},
                   dict(PARAMS["c5"]), nel=nel)


# insitu sink attributes of every config (the generators return copies)
PARAMS = {
    "c1": {"iso": "Q=0.1", "field": "velocity:mag", "view": "35,30"},
    "c2": {"iso": "temperature=0.5;Q=1.0", "slice": "y=0", "field": "temperature", "view": "-60,25"},
    "c3": {"iso": "Q=5.0", "field": "vorticity:mag", "view": "-70,20"},
    "c4": {"iso": "velocity:mag=1.2", "slice": "z=0.5", "field": "velocity:mag", "view": "+z"},
    "c5": {"iso": "Q=0.1", "field": "velocity:mag", "view": "35,30"},
}

CONFIGS = {
    "c1": lambda e0=0, e1=None, scale=1: taylor_green(e0, e1),
    "c2": lambda e0=0, e1=None, scale=1: rbc_cylinder(e0, e1, nel=(32, 32, 32 * scale)),
    "c3": lambda e0=0, e1=None, scale=1: turb_pipe(e0, e1, nel=(25, 25, 400 * scale), length=20.0 * scale),
    "c4": lambda e0=0, e1=None, scale=1: pebble_bed(e0, e1),
    # c5: `scale` is the element count of the box
    "c5": lambda e0=0, e1=None, scale=65536: c5_box(e0, e1, n_elements=scale),
}
CONFIG_ELEMENTS = {"c1": 512, "c2": 32768, "c3": 250000, "c4": 1048576, "c5": 65536}


def global_elements(name: str, scale: int = 1) -> int:
    """Elements of config `name` at `scale` (c2/c3: streamwise multiple; c5:
    the element count itself; c1/c4: fixed)."""
    if name == "c5":
        return int(scale)
    return CONFIG_ELEMENTS[name] * (scale if name in ("c2", "c3") else 1)


def make_case(name: str, rank: int = 0, nranks: int = 1, scale: int = 1) -> SemCase:
    """Partition `rank` of config `name`; `scale` multiplies the element count
    along the streamwise axis (weak scaling: scale = nranks), or is the box's
    element count for c5."""
    E = global_elements(name, scale)
    e0, e1 = partition(E, rank, nranks)
    return CONFIGS[name](e0, e1, scale)
