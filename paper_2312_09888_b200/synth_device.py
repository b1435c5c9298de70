"""Device-side generation of the large synthetic configurations (C3, C4, C5
and weak-scaled C2) -- the same formulas as synth.py, evaluated with torch on
the GPU so a 128M-537M point mesh is built in seconds instead of minutes.

Bench/test infrastructure only (the in situ path itself takes whatever device
arrays the simulation hands it).  Values match synth.py to floating-point
rounding of the transcendental functions, not bit for bit; parity checks at
these sizes therefore copy the device inputs back to the host for the oracle.
"""
from __future__ import annotations

import math

import numpy as np

from . import synth

NN = 512


def _torch():
    import torch

    return torch


def _ref_coords(nel, e0, e1, device):
    torch = _torch()
    t = torch.tensor((synth.GLL7 + 1.0) / 2.0, dtype=torch.float64, device=device)
    nx, ny, nz = nel
    e = torch.arange(e0, e1, device=device, dtype=torch.int64)
    ex, ey, ez = e % nx, (e // nx) % ny, e // (nx * ny)
    E = e1 - e0
    X = ((ex[:, None, None, None].double() + t[None, None, None, :]) / nx).expand(E, 8, 8, 8).reshape(-1)
    Y = ((ey[:, None, None, None].double() + t[None, None, :, None]) / ny).expand(E, 8, 8, 8).reshape(-1)
    Z = ((ez[:, None, None, None].double() + t[None, :, None, None]) / nz).expand(E, 8, 8, 8).reshape(-1)
    return X.contiguous(), Y.contiguous(), Z.contiguous()


def _disk(u, v):
    torch = _torch()
    return u * torch.sqrt(1.0 - 0.5 * v * v), v * torch.sqrt(1.0 - 0.5 * u * u)


class DeviceCase:
    def __init__(self, name, n_elements, e0, n_elements_global, x, y, z, fields, params):
        self.name, self.n_elements, self.e0, self.n_elements_global = name, n_elements, e0, n_elements_global
        self.x, self.y, self.z, self.fields, self.params = x, y, z, fields, params

    @property
    def n_points(self):
        return self.n_elements * NN

    def to_host(self):
        return synth.SemCase(self.name, self.n_elements, self.e0, self.n_elements_global,
                             self.x.cpu().numpy(), self.y.cpu().numpy(), self.z.cpu().numpy(),
                             {k: v.cpu().numpy() for k, v in self.fields.items()}, dict(self.params))


def rbc_cylinder(e0, e1, nel, device, seed=1):
    torch = _torch()
    X, Y, Z = _ref_coords(nel, e0, e1, device)
    x, y = _disk(2.0 * X - 1.0, 2.0 * Y - 1.0)
    z = Z
    rng = np.random.default_rng(seed)
    r = torch.hypot(x, y)
    th = torch.atan2(y, x)
    T = 1.0 - z
    for _ in range(8):
        a, m, nz_, ph = rng.uniform(0.5, 1.0), int(rng.integers(0, 5)), int(rng.integers(1, 4)), rng.uniform(0, 2 * math.pi)
        T = T + 0.05 * a * r ** m * torch.cos(m * th + ph) * torch.sin(math.pi * nz_ * z)
    vel = []
    for _ in range(3):
        acc = torch.zeros_like(x)
        for _ in range(6):
            kx, ky, kz = rng.uniform(-4, 4, size=3)
            amp, ph = rng.uniform(0.1, 0.3), rng.uniform(0, 2 * math.pi)
            acc = acc + amp * torch.sin(kx * x + ky * y + kz * z + ph)
        vel.append(acc)
    E = nel[0] * nel[1] * nel[2]
    return DeviceCase("c2", e1 - e0, e0, E, x, y, z, {"velocity": torch.stack(vel), "temperature": T[None]},
                      dict(synth.PARAMS["c2"]))


def turb_pipe(e0, e1, nel, length, device, seed=2):
    torch = _torch()
    X, Y, Z = _ref_coords(nel, e0, e1, device)
    x, y = _disk(2.0 * X - 1.0, 2.0 * Y - 1.0)
    z = length * Z
    rng = np.random.default_rng(seed)
    r2 = x * x + y * y
    vel = [torch.zeros_like(x), torch.zeros_like(x), 2.0 * (1.0 - r2)]
    damp = 1.0 - r2
    for _ in range(32):
        k = rng.uniform(-6, 6, size=3)
        amp = 0.1 * rng.uniform(0.5, 1.0, size=3)
        ph = rng.uniform(0, 2 * math.pi, size=3)
        arg = k[0] * x + k[1] * y + k[2] * z
        for c in range(3):
            vel[c] = vel[c] + amp[c] * damp * torch.sin(arg + ph[c])
    E = nel[0] * nel[1] * nel[2]
    return DeviceCase("c3", e1 - e0, e0, E, x, y, z, {"velocity": torch.stack(vel)},
                      dict(synth.PARAMS["c3"]))


def pebble_bed(e0, e1, n, device, n_spheres=146, seed=3):
    torch = _torch()
    x, y, z = _ref_coords((n, n, n), e0, e1, device)
    rng = np.random.default_rng(seed)
    cs = rng.uniform(0.1, 0.9, size=(n_spheres, 3))
    rad = rng.uniform(0.03, 0.06, size=n_spheres)
    u = torch.ones_like(x)
    v = torch.zeros_like(x)
    w = torch.zeros_like(x)
    for c, a in zip(cs, rad):
        dx, dy, dz = x - c[0], y - c[1], z - c[2]
        d2 = dx * dx + dy * dy + dz * dz + 1e-4
        d5 = d2 * d2 * torch.sqrt(d2)
        k = 0.5 * a ** 3
        u = u + k * (d2 - 3.0 * dx * dx) / d5
        v = v - k * 3.0 * dx * dy / d5
        w = w - k * 3.0 * dx * dz / d5
    return DeviceCase("c4", e1 - e0, e0, n ** 3, x, y, z, {"velocity": torch.stack([u, v, w])},
                      dict(synth.PARAMS["c4"]))


def c5_box(e0, e1, n_elements, device):
    torch = _torch()
    nel = synth.c5_lattice(n_elements)
    X, Y, Z = _ref_coords(nel, e0, e1, device)
    h = math.pi / 8.0
    x, y, z = (h * nel[0]) * X, (h * nel[1]) * Y, (h * nel[2]) * Z
    u = torch.sin(x) * torch.cos(y) * torch.cos(z)
    v = -torch.cos(x) * torch.sin(y) * torch.cos(z)
    w = torch.zeros_like(x)
    return DeviceCase("c5", e1 - e0, e0, n_elements, x, y, z, {"velocity": torch.stack([u, v, w])},
                      dict(synth.PARAMS["c5"]))


def make_case(name: str, rank: int = 0, nranks: int = 1, scale: int = 1, device="cuda", cuts=None):
    """Device partition `rank` of config `name` (see synth.make_case); `cuts`
    (nranks + 1 element indices) overrides the equal contiguous ranges."""
    E = synth.global_elements(name, scale)
    e0, e1 = (int(cuts[rank]), int(cuts[rank + 1])) if cuts is not None else synth.partition(E, rank, nranks)
    if name == "c2":
        return rbc_cylinder(e0, e1, (32, 32, 32 * scale), device)
    if name == "c3":
        return turb_pipe(e0, e1, (25, 25, 400 * scale), 20.0 * scale, device)
    if name == "c4":
        return pebble_bed(e0, e1, 128, device)
    if name == "c5":
        return c5_box(e0, e1, E, device)
    if name == "c1":
        return None
    raise KeyError(name)
