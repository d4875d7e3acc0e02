"""Seeded near-grazing facet soups for the culling stress test
(tests/test_adversarial_gpu.py). The fp32 culling hierarchy (sweep.h: chunk,
tile, member boxes — fp32 or 8-bit quantised) may only skip occluders the
exact predicate (src/geom.cpp:155-180) would reject; these scenes put the
exact decision right at its tolerances:

  * window groups: faces P (x = X) and Q (x = X + 10) face each other; a
    frame of four coplanar, edge-sharing facets at x = X + 5 leaves a small
    window around the crossing point c of the P-centroid -> Q-centroid
    sightline (all vertex-diagonal sightlines cross there too). One frame
    edge (or a corner: two edges) sits at a signed offset from c of
    0, +-1e-9, +-1e-8, +-1e-6, +-1e-4, +-1e-2 m: the pair's visibility hinges
    on a sightline grazing that edge / vertex;
  * plane groups: a facet F parallel to P at x = X + eps, eps in
    {0, 5e-10, 1e-9, 1.5e-9, 1e-8, 1e-6}, covering P: every sightline of P
    starts within eps of F's plane (the |d| <= kEps open-endpoint rule);
  * every group also rotated about z (0 and 30 degrees) and translated to
    4 km from the origin (1 m facets at km coordinates).
"""
from __future__ import annotations

import math

import numpy as np

from paper_2501_02747_b200.scenes import FacetSoup

OFFSETS = [-1e-2, -1e-4, -1e-6, -1e-8, -1e-9, 0.0, 1e-9, 1e-8, 1e-6, 1e-4, 1e-2]
EPS_PLANE = [0.0, 5e-10, 1e-9, 1.5e-9, 1e-8, 1e-6]
D = 1e-3   # the other window edges: c inside by 1 mm (other sightlines cross >= 1/16 m from c)


def _quad_x(x, y0, y1, z0, z1, plus):
    """Quad in the plane x = const, normal +x (plus) or -x (Newell, CCW from outside)."""
    if plus:
        return [(x, y0, z0), (x, y1, z0), (x, y1, z1), (x, y0, z1)]
    return [(x, y0, z0), (x, y0, z1), (x, y1, z1), (x, y1, z0)]


def _group_faces(kind, param, X, Y):
    """Faces of one group in its local frame (before rotation / translation)."""
    P = _quad_x(X, Y, Y + 1, 0.0, 1.0, True)
    Q = _quad_x(X + 10, Y, Y + 1, 0.0, 1.0, False)
    faces = [("P", P), ("Q", Q)]
    if kind == "window":
        edges, off = param     # edges: subset of "lrbt" at offset `off`, the others at +D
        cy, cz = Y + 0.5, 0.5
        o = {e: (off if e in edges else D) for e in "lrbt"}
        xf = X + 5
        wl, wr = cy - o["l"], cy + o["r"]     # window y range
        wb, wt = cz - o["b"], cz + o["t"]     # window z range
        faces += [("Fl", _quad_x(xf, Y - 1, wl, -1.0, 2.0, True)),
                  ("Fr", _quad_x(xf, wr, Y + 2, -1.0, 2.0, True)),
                  ("Fb", _quad_x(xf, wl, wr, -1.0, wb, True)),
                  ("Ft", _quad_x(xf, wl, wr, wt, 2.0, True))]
    else:
        eps = param
        faces += [("F", _quad_x(X + eps, Y - 0.5, Y + 1.5, -0.5, 1.5, False))]
    return faces


def groups():
    out = []
    for e in ["l", "r", "b", "t"]:
        for off in OFFSETS:
            out.append(("window", (e, off)))
    for corner in ["lb", "rt"]:
        for off in (-1e-9, 0.0, 1e-9, 1e-6):
            out.append(("window", (corner, off)))
    for eps in EPS_PLANE:
        out.append(("plane", eps))
    return out


def build(rotations=(0.0, 30.0), translations=((0.0, 0.0), (4000.0, 4000.0))):
    """The adversarial soup and its bookkeeping: per group the face indices of
    P and Q (and the frame / F), plus the stressed sightlines and sources."""
    ids, rings, meta = [], [], []
    gi = 0
    for rot in rotations:
        th = math.radians(rot)
        c, s = math.cos(th), math.sin(th)
        for tx, ty in translations:
            for kind, param in groups():
                # local frame: groups 20 m apart in y, rotated about the group's
                # own P corner, then translated
                X0, Y0 = 0.0, 20.0 * gi
                faces = _group_faces(kind, param, 0.0, 0.0)
                first = len(ids)
                for name, ring in faces:
                    pts = []
                    for (x, y, z) in ring:
                        xr, yr = c * x - s * y, s * x + c * y
                        pts.append((xr + X0 + tx, yr + Y0 + ty, z))
                    ids.append(f"G{gi}_{name}")
                    rings.append(pts)
                meta.append({"kind": kind, "param": param, "rot": rot, "translate": (tx, ty),
                             "faces": list(range(first, len(ids))), "origin": (X0 + tx, Y0 + ty),
                             "rotc": (c, s)})
                gi += 1
    off = np.zeros(len(rings) + 1, np.int32)
    off[1:] = np.cumsum([len(r) for r in rings])
    soup = FacetSoup(ids=ids, vert_off=off, verts=np.array([p for r in rings for p in r], np.float64),
                     name="adversarial")
    return soup, meta


def _to_world(m, x, y, z):
    c, s = m["rotc"]
    X0, Y0 = m["origin"]
    return (c * x - s * y + X0, s * x + c * y + Y0, z)


def stressed_segments(meta):
    """Per group: the P-centroid -> Q-centroid sightline, the two diagonals of
    P and Q's vertices through c, and P-centroid -> points of Q near the window
    edge (offset by 0, 1e-12, 1e-10 m either side)."""
    A, B = [], []
    for m in meta:
        pc = _to_world(m, 0.0, 0.5, 0.5)
        for q in [(10.0, 0.5, 0.5)] + [(10.0, 0.5 + d, 0.5) for d in (1e-12, -1e-12, 1e-10, -1e-10, 2e-9, -2e-9)]:
            A.append(pc)
            B.append(_to_world(m, *q))
        A.append(_to_world(m, 0.0, 0.0, 0.0))
        B.append(_to_world(m, 10.0, 1.0, 1.0))
        A.append(_to_world(m, 0.0, 1.0, 0.0))
        B.append(_to_world(m, 10.0, 0.0, 1.0))
    return np.array(A, np.float64), np.array(B, np.float64)


def sources(meta):
    """Two region sources per group: on the c line between P and the frame,
    and behind P."""
    out = []
    for m in meta:
        out.append(_to_world(m, 2.5, 0.5, 0.5))
        out.append(_to_world(m, -3.0, 0.5, 0.5))
    return np.array(out, np.float64)
