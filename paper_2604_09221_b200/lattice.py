"""Lattice geometry of d times the standard triangle (host side, once per T).

Conventions follow the reference so indices, fingerprints and reports line
up byte for byte:

* point order: ``(i, j)`` for ``i`` in ``0..d`` and ``j`` in ``0..d-i``
  (reference lattice.py:30-37); the index of ``(i, j)`` is
  ``i*(d+1) - i*(i-1)/2 + j``;
* ``harnack_bound(d) = (d-1)(d-2)/2 + 1`` (lattice.py:53-55);
* ``Triangulation.fingerprint()`` is the sha256 of the compact JSON
  ``{"degree": d, "edges": sorted(edges)}`` (lattice.py:107-113).

Validation here is an independent implementation: range and degeneracy
checks, exact pairwise crossing / T-joint tests (vectorised int64), then a
face check by area: every empty lattice 3-cycle of the edge graph is a
face, and the faces must tile the doubled area d^2.
"""

from __future__ import annotations

import hashlib
import json
from dataclasses import dataclass

import numpy as np

from .errors import InvalidDegree, NotATriangulation, NotUnimodular, PointOutOfRange

Point = tuple[int, int]
Edge = tuple[Point, Point]


def lattice_points(d: int) -> list[Point]:
    if d < 1:
        raise InvalidDegree(f"degree must be >= 1, got {d}")
    return [(i, j) for i in range(d + 1) for j in range(d + 1 - i)]


def num_points(d: int) -> int:
    return (d + 1) * (d + 2) // 2


def point_index(d: int) -> dict[Point, int]:
    return {p: k for k, p in enumerate(lattice_points(d))}


def index_of(d: int, i: int, j: int) -> int:
    """Canonical index of (i, j) without building the dictionary."""
    return i * (d + 1) - i * (i - 1) // 2 + j


def num_edges_unimodular(d: int) -> int:
    return (3 * d * d + 3 * d) // 2


def harnack_bound(d: int) -> int:
    return (d - 1) * (d - 2) // 2 + 1


def _doubled_area(a: Point, b: Point, c: Point) -> int:
    return abs((b[0] - a[0]) * (c[1] - a[1]) - (b[1] - a[1]) * (c[0] - a[0]))


def normalize_edge(p: Point, q: Point) -> Edge:
    return (p, q) if p <= q else (q, p)


@dataclass(frozen=True)
class Triangulation:
    """Edges (sorted, normalised) plus triangles (sorted vertex triples)."""

    degree: int
    edges: tuple[Edge, ...]
    triangles: tuple[tuple[Point, Point, Point], ...]

    @property
    def edge_set(self) -> frozenset[Edge]:
        return frozenset(self.edges)

    def points_used(self) -> set[Point]:
        return {p for e in self.edges for p in e}

    @property
    def is_unimodular(self) -> bool:
        d = self.degree
        return (
            len(self.edges) == num_edges_unimodular(d)
            and len(self.triangles) == d * d
            and len(self.points_used()) == num_points(d)
            and all(_doubled_area(*t) == 1 for t in self.triangles)
        )

    def fingerprint(self) -> str:
        payload = json.dumps(
            {"degree": self.degree, "edges": sorted(self.edges)}, separators=(",", ":")
        )
        return hashlib.sha256(payload.encode()).hexdigest()


def fingerprint_of(T) -> str:
    """Fingerprint of any triangulation-like object (``.degree``, ``.edges``)."""
    fp = getattr(T, "fingerprint", None)
    if callable(fp):
        return fp()
    payload = json.dumps(
        {"degree": int(T.degree), "edges": sorted(_norm_edges(T.edges))},
        separators=(",", ":"),
    )
    return hashlib.sha256(payload.encode()).hexdigest()


def _norm_edges(edges) -> list[Edge]:
    out = []
    for p, q in edges:
        p = (int(p[0]), int(p[1]))
        q = (int(q[0]), int(q[1]))
        out.append(normalize_edge(p, q))
    return out


def _orient(px, py, qx, qy, rx, ry):
    return (qx - px) * (ry - py) - (qy - py) * (rx - px)


def _check_planar(edges: list[Edge]) -> None:
    a = np.array([e[0] for e in edges], dtype=np.int64)
    b = np.array([e[1] for e in edges], dtype=np.int64)
    ax, ay, bx, by = a[:, 0], a[:, 1], b[:, 0], b[:, 1]
    # proper crossings: both segments straddle each other's supporting line
    s1 = np.sign(_orient(ax[:, None], ay[:, None], bx[:, None], by[:, None], ax[None], ay[None]))
    s2 = np.sign(_orient(ax[:, None], ay[:, None], bx[:, None], by[:, None], bx[None], by[None]))
    cross = (s1 * s2 < 0) & (s1.T * s2.T < 0)
    if cross.any():
        i, j = np.argwhere(cross)[0]
        raise NotATriangulation(f"edges {edges[i]} and {edges[j]} cross")
    verts = np.array(sorted({p for e in edges for p in e}), dtype=np.int64)
    vx, vy = verts[:, 0], verts[:, 1]
    col = _orient(ax[:, None], ay[:, None], bx[:, None], by[:, None], vx[None], vy[None]) == 0
    inside = ((vx[None] - ax[:, None]) * (vx[None] - bx[:, None])
              + (vy[None] - ay[:, None]) * (vy[None] - by[:, None])) < 0
    bad = col & inside
    if bad.any():
        i, j = np.argwhere(bad)[0]
        raise NotATriangulation(
            f"point {tuple(int(x) for x in verts[j])} lies inside edge {edges[i]}"
        )


def _faces(d: int, edges: list[Edge]) -> list[tuple[Point, Point, Point]]:
    """Empty 3-cycles of a planar straight-line lattice graph (its triangular faces)."""
    nbr: dict[Point, set[Point]] = {}
    for p, q in edges:
        nbr.setdefault(p, set()).add(q)
        nbr.setdefault(q, set()).add(p)
    verts = sorted(nbr)
    tris = set()
    for p, q in edges:
        for r in nbr[p] & nbr[q]:
            t = tuple(sorted((p, q, r)))
            if t in tris or _doubled_area(*t) == 0:
                continue
            # a 3-cycle of a PSLG is a face iff no vertex lies strictly inside
            a, b, c = t
            s = 1 if _orient(*a, *b, *c) > 0 else -1
            empty = True
            for v in verts:
                if v in t:
                    continue
                if (s * _orient(*a, *b, *v) > 0 and s * _orient(*b, *c, *v) > 0
                        and s * _orient(*c, *a, *v) > 0):
                    empty = False
                    break
            if empty:
                tris.add(t)
    return sorted(tris)


def validate_triangulation(d: int, edges, require_unimodular: bool = True) -> Triangulation:
    """Check an edge list and return the triangulation with its triangles."""
    if d < 1:
        raise InvalidDegree(f"degree must be >= 1, got {d}")
    norm: set[Edge] = set()
    for p, q in edges:
        p, q = (int(p[0]), int(p[1])), (int(q[0]), int(q[1]))
        for pt in (p, q):
            if pt[0] < 0 or pt[1] < 0 or pt[0] + pt[1] > d:
                raise PointOutOfRange(f"point {pt} outside degree-{d} lattice")
        if p == q:
            raise NotATriangulation(f"degenerate edge at {p}")
        norm.add(normalize_edge(p, q))
    if not norm:
        raise NotATriangulation("empty edge list")
    edge_list = sorted(norm)
    _check_planar(edge_list)
    tris = _faces(d, edge_list)
    area = sum(_doubled_area(*t) for t in tris)
    if area != d * d:
        raise NotATriangulation(
            f"subdivision does not cover the degree-{d} triangle "
            f"(covered doubled area {area} of {d * d})"
        )
    T = Triangulation(d, tuple(edge_list), tuple(tris))
    if require_unimodular and not T.is_unimodular:
        raise NotUnimodular(
            f"{len(edge_list)} edges, {len(tris)} triangles, "
            f"{len(T.points_used())} of {num_points(d)} points used"
        )
    return T


def staircase(d: int) -> Triangulation:
    """The staircase (Harnack) triangulation: unit edges along (1,0), (0,1), (1,-1).

    It is the projection of the lifting i^2 + i*j + j^2, i.e. the reference's
    ``builtin("delaunay-d")`` (builtins.py:30-38); tests pin the equality.
    """
    if d < 1:
        raise InvalidDegree(f"degree must be >= 1, got {d}")
    edges = set()
    tris = set()
    for i in range(d + 1):
        for j in range(d + 1 - i):
            if i + j + 1 <= d:
                edges.add(((i, j), (i + 1, j)))
                edges.add(((i, j), (i, j + 1)))
                edges.add(normalize_edge((i + 1, j), (i, j + 1)))
                tris.add(tuple(sorted(((i, j), (i + 1, j), (i, j + 1)))))
            if i + j + 2 <= d:
                tris.add(tuple(sorted(((i + 1, j), (i, j + 1), (i + 1, j + 1)))))
    return Triangulation(d, tuple(sorted(edges)), tuple(sorted(tris)))


# ---------------------------------------------------------------------------
# the order-6 symmetry group of the triangle acting on barycentric coordinates


@dataclass(frozen=True)
class SymmetryElement:
    name: str
    perm: tuple[int, int, int]

    def apply(self, d: int, p: Point) -> Point:
        c = (p[0], p[1], d - p[0] - p[1])
        return (c[self.perm[0]], c[self.perm[1]])


SYMMETRY_GROUP = (
    SymmetryElement("e", (0, 1, 2)),
    SymmetryElement("r", (2, 0, 1)),
    SymmetryElement("rr", (1, 2, 0)),
    SymmetryElement("t", (1, 0, 2)),
    SymmetryElement("tr", (2, 1, 0)),
    SymmetryElement("trr", (0, 2, 1)),
)
TRANSPOSE = SYMMETRY_GROUP[3]


def map_triangulation(T, g: SymmetryElement) -> Triangulation:
    d = T.degree
    edges = tuple(sorted(normalize_edge(g.apply(d, p), g.apply(d, q)) for p, q in T.edges))
    tris = tuple(
        sorted(tuple(sorted(g.apply(d, p) for p in t)) for t in getattr(T, "triangles", ()))
    )
    return Triangulation(d, edges, tris)
