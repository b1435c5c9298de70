"""ctypes front-end of the C oracle (sem_oracle.c) plus an independent numpy
restatement of the derived fields.  TEST INFRASTRUCTURE ONLY (see
oracle/__init__.py).

Two independent CPU formulations exist on purpose:
  * `libsem_oracle.so` restates the GPU algorithm operation for operation
    (explicit fma, same order): the GPU must match it BIT-EXACTLY (Q,
    vorticity, case indices, triangle vertices, image keys, RGBA).
  * `derived_numpy` computes the same calculus with einsum/vectorised numpy
    (different summation order, no fma): it pins the C oracle's mathematics
    to within the north star's 1e-12 (norm-relative) without sharing code.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "build", "libsem_oracle.so")

SRC_Q, SRC_WMAG, SRC_UMAG, SRC_SCALAR0, SRC_SCALAR1, SRC_PLANE = 0, 1, 2, 3, 4, 8
DEFAULT_ANCHORS = ((0.0, (59, 76, 192)), (0.5, (255, 255, 255)), (1.0, (180, 4, 38)))


def build(force: bool = False) -> str:
    src = [os.path.join(HERE, f) for f in ("sem_oracle.c", "mc_tables.h", "Makefile")]
    if force or not os.path.exists(LIB) or any(os.path.getmtime(s) > os.path.getmtime(LIB) for s in src):
        subprocess.run(["make", "-s", "-C", HERE, "-B" if force else "build/libsem_oracle.so"], check=True)
    return LIB


class OrcFields(C.Structure):
    _fields_ = [
        ("E", C.c_int64),
        ("x", C.c_void_p), ("y", C.c_void_p), ("z", C.c_void_p),
        ("u", C.c_void_p), ("v", C.c_void_p), ("w", C.c_void_p),
        ("s0", C.c_void_p), ("s1", C.c_void_p),
        ("n_surf", C.c_int),
        ("surf_src", C.c_int * 4),
        ("surf_iso", C.c_double * 4),
        ("surf_n", (C.c_double * 3) * 4),
        ("color_src", C.c_int),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = C.CDLL(LIB)
        vp, i64 = C.c_void_p, C.c_int64
        L.orc_gll.argtypes = [C.c_int, vp, vp]
        L.orc_derived.argtypes = [C.POINTER(OrcFields), i64, i64, vp, vp, vp, vp]
        L.orc_mc.argtypes = [C.POINTER(OrcFields), i64, i64, vp, vp, i64, vp, vp, vp]
        L.orc_mc.restype = i64
        L.orc_raster.argtypes = [vp, i64, vp, C.c_int, C.c_int, vp]
        L.orc_zbuf_clear.argtypes = [vp, i64]
        L.orc_composite_min.argtypes = [vp, vp, i64]
        L.orc_colormap.argtypes = [C.c_int, vp, vp, vp, i64, vp]
        L.orc_resolve.argtypes = [vp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, vp, vp, vp, vp, vp]
        L.orc_render_structured.argtypes = [C.c_int, vp, vp, i64, C.c_int, C.c_int, C.c_int, C.c_int,
                                            C.c_double, C.c_double, vp, vp]
        L.orc_pipeline_mt.argtypes = [C.c_int, C.POINTER(OrcFields), vp, C.c_int, C.c_int, C.c_double,
                                      C.c_double, C.c_int, vp, vp, vp, vp, vp, vp]
        L.orc_pipeline_mt.restype = i64
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def gll(order: int = 7):
    x = np.zeros(order + 1)
    D = np.zeros((order + 1, order + 1))
    assert lib().orc_gll(order, x.ctypes.data, D.ctypes.data) == 0
    return x, D


class CaseFields:
    """Host arrays of one SEM partition plus the source mapping of a
    pipeline -- mirrors the product's name resolution (abi.cu resolve_src)."""

    def __init__(self, x, y, z, fields: dict, velocity: str = "velocity"):
        self.x, self.y, self.z = (np.ascontiguousarray(a, dtype=np.float64) for a in (x, y, z))
        self.E = self.x.size // 512
        self.fields = {k: np.ascontiguousarray(np.asarray(v, dtype=np.float64).reshape(-1, self.x.size))
                       for k, v in fields.items()}
        self.velocity = velocity
        self._scalars: list[str] = []

    def src(self, name: str) -> int:
        if name == "Q":
            return SRC_Q
        if name == "vorticity:mag":
            return SRC_WMAG
        if name.endswith(":mag"):
            if name[:-4] != self.velocity:
                raise ValueError("':mag' only for the velocity field")
            return SRC_UMAG
        if name not in self.fields:
            raise KeyError(name)
        if self.fields[name].shape[0] != 1:
            raise ValueError(f"field {name!r} has {self.fields[name].shape[0]} components")
        if name not in self._scalars:
            self._scalars.append(name)
        return SRC_SCALAR0 + self._scalars.index(name)

    def native(self, surfaces=(), color: str | None = None) -> OrcFields:
        """surfaces: sequence of ('iso', field, value) or ('slice', (nx,ny,nz), c)."""
        f = OrcFields()
        f.E = self.E
        f.x, f.y, f.z = _p(self.x), _p(self.y), _p(self.z)
        vel = self.fields.get(self.velocity)
        if vel is not None:
            f.u, f.v, f.w = vel[0].ctypes.data, vel[1].ctypes.data, vel[2].ctypes.data
        self._scalars = []
        f.n_surf = len(surfaces)
        for k, s in enumerate(surfaces):
            if s[0] == "iso":
                f.surf_src[k] = self.src(s[1])
                f.surf_iso[k] = float(s[2])
            else:
                f.surf_src[k] = SRC_PLANE + k
                f.surf_iso[k] = float(s[2])
                for a in range(3):
                    f.surf_n[k][a] = float(s[1][a])
        f.color_src = self.src(color) if color is not None else -1
        arrs = [self.fields[n][0] for n in self._scalars]
        if len(arrs) > 0:
            f.s0 = arrs[0].ctypes.data
        if len(arrs) > 1:
            f.s1 = arrs[1].ctypes.data
        self._keep = arrs
        return f


def derived(cf: CaseFields):
    """(Q, |w|, vorticity AoS, |u|) for every node, C oracle."""
    n = cf.x.size
    q, wm, um = np.empty(n), np.empty(n), np.empty(n)
    vort = np.empty(3 * n)
    f = cf.native()
    lib().orc_derived(C.byref(f), 0, cf.E, _p(q), _p(wm), _p(vort), _p(um))
    return q, wm, vort, um


def mc(cf: CaseFields, surfaces, color: str, cases: bool = False):
    """Triangles (n, 3, 4) float32, meta (n,) uint64, colour range, [cases (E, 343) uint32]."""
    f = cf.native(surfaces, color)
    cmin, cmax = C.c_double(), C.c_double()
    n = lib().orc_mc(C.byref(f), 0, cf.E, None, None, 0, C.byref(cmin), C.byref(cmax), None)
    tri = np.empty((max(n, 1), 3, 4), np.float32)
    meta = np.empty(max(n, 1), np.uint64)
    cs = np.empty((cf.E, 343), np.uint32) if cases else None
    f = cf.native(surfaces, color)
    lib().orc_mc(C.byref(f), 0, cf.E, _p(tri), _p(meta), n, None, None, _p(cs))
    out = (tri[:n], meta[:n], (cmin.value, cmax.value))
    return out + ((cs,) if cases else ())


def _view16(view, persp=None) -> np.ndarray:
    """3x4 view rows + perspective row (zeros = orthographic), as orc_raster takes them."""
    v = np.zeros(16)
    a = np.asarray(view, dtype=np.float64).ravel()
    v[:a.size] = a                                  # 12 values, or 16 with the perspective row
    if persp is not None:
        v[12:] = np.asarray(persp, dtype=np.float64)
    return v


def raster(tri: np.ndarray, view, W: int, H: int, zbuf: np.ndarray | None = None, persp=None) -> np.ndarray:
    t = np.ascontiguousarray(tri, dtype=np.float32)
    V = _view16(view, persp)
    if zbuf is None:
        zbuf = np.empty(W * H, np.uint64)
        lib().orc_zbuf_clear(_p(zbuf), W * H)
    lib().orc_raster(_p(t), t.shape[0], _p(V), W, H, _p(zbuf))
    return zbuf


def composite_min(dst: np.ndarray, src: np.ndarray) -> np.ndarray:
    lib().orc_composite_min(_p(dst), _p(src), dst.size)
    return dst


def _anchors(anchors):
    if tuple(anchors) == DEFAULT_ANCHORS:
        return 0, None, None
    ts = np.array([a[0] for a in anchors], np.float64)
    rgb = np.array([a[1] for a in anchors], np.uint8).ravel()
    return len(anchors), ts, rgb


def resolve(zbuf, W, H, lo, hi, anchors=DEFAULT_ANCHORS, bg=(0, 0, 0, 0)):
    n, ts, rgb = _anchors(anchors)
    out = np.empty((H, W, 4), np.uint8)
    dep = np.empty((H, W), np.float32)
    b = np.array(bg, np.uint8)
    lib().orc_resolve(_p(zbuf), W, H, float(lo), float(hi), n, _p(ts), _p(rgb), _p(b), _p(out), _p(dep))
    return out, dep


def colormap(t: np.ndarray, anchors=DEFAULT_ANCHORS) -> np.ndarray:
    n, ts, rgb = _anchors(anchors)
    tt = np.ascontiguousarray(t, dtype=np.float64).ravel()
    out = np.empty((tt.size, 3), np.uint8)
    lib().orc_colormap(n, _p(ts), _p(rgb), _p(tt), tt.size, _p(out))
    return out.reshape(np.shape(t) + (3,))


def render_structured(blocks, rows: int, comps: int, mode: int, W: int, H: int, vmin=None, vmax=None):
    """blocks: list of (values AoS float64, ni)."""
    keep = [np.ascontiguousarray(v, dtype=np.float64) for v, _ in blocks]
    ptrs = (C.c_void_p * len(keep))(*[k.ctypes.data for k in keep])
    nis = (C.c_int64 * len(keep))(*[int(n) for _, n in blocks])
    rgb = np.empty(W * H * 3, np.uint8)
    rng = np.empty(2)
    lib().orc_render_structured(len(keep), C.addressof(ptrs), C.addressof(nis), rows, comps, mode, W, H,
                                math.nan if vmin is None else float(vmin),
                                math.nan if vmax is None else float(vmax), _p(rgb), _p(rng))
    return rgb.tobytes(), (float(rng[0]), float(rng[1]))


def pipeline_mt(cf: CaseFields, surfaces, color, view, W, H, nthreads: int, vmin=None, vmax=None,
                anchors=DEFAULT_ANCHORS, bg=(0, 0, 0, 0), persp=None):
    """Full step on `nthreads` CPU threads -> (rgba, depth, ntri, range)."""
    f = cf.native(surfaces, color)
    n, ts, rgb = _anchors(anchors)
    V = _view16(view, persp)
    out = np.empty((H, W, 4), np.uint8)
    dep = np.empty((H, W), np.float32)
    b = np.array(bg, np.uint8)
    rng = np.empty(2)
    ntri = lib().orc_pipeline_mt(int(nthreads), C.byref(f), _p(V), W, H,
                                 math.nan if vmin is None else float(vmin),
                                 math.nan if vmax is None else float(vmax),
                                 n, _p(ts), _p(rgb), _p(b), _p(out), _p(dep), _p(rng))
    return out, dep, int(ntri), (float(rng[0]), float(rng[1]))


# ---------------------------------------------------------------------------
# independent numpy formulation (no fma, einsum order) for the 1e-12 check
# ---------------------------------------------------------------------------

def derived_numpy(x, y, z, u, v, w, D=None):
    """Q, vorticity (3, n), |u| by textbook formulas: J = d(x,y,z)/d(r,s,t),
    grad u = (du/dr) J^-1, Q = 1/2 (|Omega|^2 - |S|^2)."""
    if D is None:
        _, D = gll(7)
    E = np.asarray(x).size // 512

    def dd(f):
        f = np.asarray(f, dtype=np.float64).reshape(E, 8, 8, 8)   # [e, k, j, i]
        fr = np.einsum("im,ekjm->ekji", D, f)
        fs = np.einsum("jm,ekmi->ekji", D, f)
        ft = np.einsum("km,emji->ekji", D, f)
        return np.stack([fr, fs, ft], axis=-1).reshape(-1, 3)     # (n, 3): d/dr, d/ds, d/dt

    Jx, Jy, Jz = dd(x), dd(y), dd(z)
    J = np.stack([Jx, Jy, Jz], axis=1)                            # (n, 3 [x,y,z], 3 [r,s,t])
    Jinv = np.linalg.inv(J)                                       # (n, 3 [r,s,t], 3 [x,y,z])
    Ur = np.stack([dd(u), dd(v), dd(w)], axis=1)                  # (n, 3 [u,v,w], 3 [r,s,t])
    A = np.einsum("nad,ndb->nab", Ur, Jinv)                       # A[a][b] = du_a/dx_b
    S = 0.5 * (A + np.transpose(A, (0, 2, 1)))
    O = 0.5 * (A - np.transpose(A, (0, 2, 1)))
    Q = 0.5 * (np.sum(O * O, axis=(1, 2)) - np.sum(S * S, axis=(1, 2)))
    vort = np.stack([A[:, 2, 1] - A[:, 1, 2], A[:, 0, 2] - A[:, 2, 0], A[:, 1, 0] - A[:, 0, 1]])
    umag = np.sqrt(np.asarray(u) ** 2 + np.asarray(v) ** 2 + np.asarray(w) ** 2)
    gradnorm2 = np.sum(A * A, axis=(1, 2))
    return Q, vort, umag.ravel(), gradnorm2


def dssum(gid: np.ndarray, vals: np.ndarray, rank_lo=None) -> np.ndarray:
    """Direct stiffness average (test oracle for nkb_dssum, dssum.cu header).

    gid/vals: global arrays in rank order; rank_lo: first global index of
    every rank (default: one rank).  For a global id with copies on ranks
    r0 < r1 < ...: P_r = left fold of rank r's copies in increasing index,
    total = ((P_r0 + P_r1) + ...), and every copy becomes total / count.
    Plain float64 numpy arithmetic (IEEE, no FMA), vectorised over ids."""
    gid = np.asarray(gid, dtype=np.int64)
    v = np.asarray(vals, dtype=np.float64)
    n = v.size
    rank = np.zeros(n, np.int64) if rank_lo is None else np.searchsorted(np.asarray(rank_lo), np.arange(n), "right") - 1
    order = np.argsort(gid, kind="stable")                 # copies of an id in increasing global index
    g = gid[order]
    start = np.flatnonzero(np.r_[True, g[1:] != g[:-1]])
    count = np.diff(np.r_[start, n])
    part = v[order[start]].copy()                          # running partial of the current rank
    prank = rank[order[start]].copy()
    total = np.zeros_like(part)
    have = np.zeros(part.size, bool)
    for k in range(1, int(count.max())):
        live = count > k
        idx = order[start[live] + k]
        same = rank[idx] == prank[live]
        li = np.flatnonzero(live)
        a = li[same]                                       # same rank: extend the partial
        part[a] = part[a] + v[idx[same]]
        b = li[~same]                                      # next rank: close the partial
        total[b] = np.where(have[b], total[b] + part[b], part[b])
        have[b] = True
        part[b] = v[idx[~same]]
        prank[b] = rank[idx[~same]]
    total = np.where(have, total + part, part)
    avg = total / count
    out = np.empty_like(v)
    out[order] = np.repeat(avg, count)
    return out
