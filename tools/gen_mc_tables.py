#!/usr/bin/env python3
"""Generate the marching-cubes case tables used by BOTH the CUDA kernels and
the CPU oracle.

Neither the reference (`/root/reference`, pure Python, structured 2D only --
SPEC.md:76, :347) nor the paper ships a triangle table, and the classic
Lorensen/Bourke table is third-party data we do not vendor.  So the table is
*derived* here from first principles, deterministically:

* cube vertices in VTK_HEXAHEDRON order: v0 (0,0,0) v1 (1,0,0) v2 (1,1,0)
  v3 (0,1,0) v4 (0,0,1) v5 (1,0,1) v6 (1,1,1) v7 (0,1,1);
* edges oriented lower-vertex-first (so a vertex on a shared edge is computed
  identically by every sub-hex that owns the edge);
* a corner is INSIDE when scalar >= iso (the case bit v is set);
* on every face the crossed edges are paired into segments; an ambiguous face
  (4 crossings, diagonal corners inside) separates the inside corners.  The
  rule depends only on the face's own corner states, so two sub-hexes that
  share a face make the same choice and the surface is crack-free;
* segments are oriented with the inside region on their left when the face is
  viewed from outside the cube, chained into closed loops, and each loop is
  fan-triangulated from the first vertex whose fan has no diagonal lying in
  a cube face (so neighbouring sub-hexes never stack triangles on a shared
  face segment); triangle normals (right-hand rule) point from the inside
  region to the outside.

Output: the same text to `paper_2312_09888_b200/csrc/mc_tables.h` (product)
and `oracle/mc_tables.h` (checker).  `tests/test_mc_tables.py` checks the two
files are byte-identical and that the table is closed/consistent.
"""
from __future__ import annotations

import os
import sys

import numpy as np

VERTS = np.array(
    [(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0), (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1)],
    dtype=float,
)
# edges, endpoint with the lower lattice node index (i + 8j + 64k) first
EDGES = [(0, 1), (1, 2), (3, 2), (0, 3), (4, 5), (5, 6), (7, 6), (4, 7), (0, 4), (1, 5), (2, 6), (3, 7)]
# faces: cyclic vertex order + outward normal
FACES = [
    ((0, 1, 2, 3), (0, 0, -1)),
    ((4, 5, 6, 7), (0, 0, 1)),
    ((0, 1, 5, 4), (0, -1, 0)),
    ((3, 2, 6, 7), (0, 1, 0)),
    ((0, 3, 7, 4), (-1, 0, 0)),
    ((1, 2, 6, 5), (1, 0, 0)),
]


def edge_id(a: int, b: int) -> int:
    for i, (p, q) in enumerate(EDGES):
        if {p, q} == {a, b}:
            return i
    raise KeyError((a, b))


def mid(e: int) -> np.ndarray:
    a, b = EDGES[e]
    return 0.5 * (VERTS[a] + VERTS[b])


def case_polygons(mask: int) -> list[list[int]]:
    inside = [(mask >> v) & 1 == 1 for v in range(8)]
    segs: list[tuple[int, int]] = []
    for fv, fn in FACES:
        n = np.array(fn, dtype=float)
        fe = [edge_id(fv[i], fv[(i + 1) % 4]) for i in range(4)]  # edge i joins fv[i], fv[i+1]
        crossed = [inside[fv[i]] != inside[fv[(i + 1) % 4]] for i in range(4)]
        pairs: list[tuple[int, int, np.ndarray]] = []
        nc = sum(crossed)
        if nc == 0:
            continue
        if nc == 2:
            a, b = [i for i in range(4) if crossed[i]]
            ins = [VERTS[v] for v in fv if inside[v]]
            c = np.mean(ins, axis=0)
            pairs.append((fe[a], fe[b], c))
        elif nc == 4:
            # ambiguous face: separate each inside corner
            for i in range(4):
                if inside[fv[i]]:
                    # corner fv[i] lies between edges (i-1) and i
                    pairs.append((fe[(i - 1) % 4], fe[i], VERTS[fv[i]]))
        else:
            raise AssertionError("odd crossing count on a face")
        for ea, eb, c in pairs:
            p, q = mid(ea), mid(eb)
            if np.dot(n, np.cross(q - p, c - p)) > 0:
                segs.append((ea, eb))
            else:
                segs.append((eb, ea))
    # chain segments into loops
    nxt: dict[int, int] = {}
    for a, b in segs:
        assert a not in nxt, (mask, segs)
        nxt[a] = b
    assert sorted(nxt.keys()) == sorted(nxt.values())
    loops: list[list[int]] = []
    seen: set[int] = set()
    for start in sorted(nxt.keys()):
        if start in seen:
            continue
        loop = [start]
        seen.add(start)
        e = nxt[start]
        while e != start:
            loop.append(e)
            seen.add(e)
            e = nxt[e]
        loops.append(loop)
    return loops


def _share_face(e1: int, e2: int) -> bool:
    va, vb = set(EDGES[e1]), set(EDGES[e2])
    return any(va <= set(fv) and vb <= set(fv) for fv, _ in FACES)


def _fan_start(loop: list[int]) -> int:
    """First loop vertex whose fan has no diagonal lying in a cube face.

    A diagonal between two crossing points of the same face would lie in
    that face; the neighbouring sub-hex can make the same choice from its
    side, giving four triangles on one segment (a non-manifold seam).
    """
    n = len(loop)
    for s0 in range(n):
        diags = [loop[(s0 + i) % n] for i in range(2, n - 1)]
        if not any(_share_face(loop[s0], d) for d in diags):
            return s0
    raise AssertionError(f"no face-free fan for loop {loop}")


def case_triangles(mask: int) -> list[tuple[int, int, int]]:
    tris = []
    for loop in case_polygons(mask):
        s0 = _fan_start(loop)
        lp = loop[s0:] + loop[:s0]
        for i in range(1, len(lp) - 1):
            tris.append((lp[0], lp[i], lp[i + 1]))
    return tris


def build():
    tables = [case_triangles(m) for m in range(256)]
    # orientation convention: normal points from inside to outside.  Check on
    # the single-corner case v0 (inside at the origin corner).
    t = tables[1][0]
    nrm = np.cross(mid(t[1]) - mid(t[0]), mid(t[2]) - mid(t[0]))
    flip = np.dot(nrm, (1, 1, 1)) < 0
    if flip:
        tables = [[(a, c, b) for (a, b, c) in tl] for tl in tables]
    return tables


def render_header(tables) -> str:
    maxt = max(len(t) for t in tables)
    ntri = ",".join(str(len(t)) for t in tables)
    tri_rows = []
    for tl in tables:
        flat = [e for t in tl for e in t] + [-1] * (3 * maxt - 3 * len(tl))
        tri_rows.append("{" + ",".join(str(e) for e in flat) + "}")
    lines = [
        "/* GENERATED by tools/gen_mc_tables.py -- do not edit.",
        " * Marching-cubes case tables (VTK_HEXAHEDRON vertex order, inside = s >= iso,",
        " * ambiguous faces separate inside corners, normals point inside -> outside).",
        " * Shared verbatim by the CUDA kernels (csrc/) and the CPU oracle (oracle/).",
        " * The *_DATA macros let device code define its own copies. */",
        "#ifndef NKB_MC_TABLES_H",
        "#define NKB_MC_TABLES_H",
        f"#define NKB_MC_MAX_TRI {maxt}",
        "/* edge e joins cube vertices EDGE_V[e][0] (lower lattice node id) and [1] */",
        "#define NKB_MC_EDGE_V_DATA " + ", ".join(f"{{{a},{b}}}" for a, b in EDGES),
        "/* vertex v sits at lattice offset (di, dj, dk) = VERT_OFF[v] */",
        "#define NKB_MC_VERT_OFF_DATA " + ", ".join("{%d,%d,%d}" % tuple(int(x) for x in v) for v in VERTS),
        "/* number of triangles of case c */",
        "#define NKB_MC_NTRI_DATA " + ntri,
        "/* triangle k of case c uses edges TRI[c][3k..3k+2]; unused = -1 */",
        "#define NKB_MC_TRI_DATA \\",
    ]
    for i, r in enumerate(tri_rows):
        lines.append("  " + r + ("," if i < 255 else "") + (" \\" if i < 255 else ""))
    lines += [
        "#ifndef NKB_MC_NO_HOST_TABLES",
        "static const unsigned char nkb_mc_edge_v[12][2] = {NKB_MC_EDGE_V_DATA};",
        "static const unsigned char nkb_mc_vert_off[8][3] = {NKB_MC_VERT_OFF_DATA};",
        "static const unsigned char nkb_mc_ntri[256] = {NKB_MC_NTRI_DATA};",
        f"static const signed char nkb_mc_tri[256][{3 * maxt}] = {{NKB_MC_TRI_DATA}};",
        "#endif",
        "#endif",
    ]
    return "\n".join(lines) + "\n"


def main(argv):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    text = render_header(build())
    outs = [
        os.path.join(root, "paper_2312_09888_b200", "csrc", "mc_tables.h"),
        os.path.join(root, "oracle", "mc_tables.h"),
    ]
    for p in outs:
        os.makedirs(os.path.dirname(p), exist_ok=True)
        with open(p, "w") as f:
            f.write(text)
    print("wrote", *outs)


if __name__ == "__main__":
    main(sys.argv)
