"""The reflected triangulation on the diamond |i| + |j| <= d (host side).

Same complex, vertex numbering and edge order as the reference
(diamond.py:25-105), because that numbering is what the C ABI descriptor
carries and what the reference kernel's check order follows:

* vertices: lexicographic points of the diamond (diamond.py:25-31);
* edges: the four sign reflections of T's edges, deduplicated, as sorted
  ``(u, v)`` index pairs with ``u < v`` (diamond.py:80-92);
* antipodal pairs: boundary points ``p`` with ``p > -p`` that are used by
  some edge, as ``(index(-p), index(p))`` sorted (diamond.py:94-98);
* sign extension: ``src[v]`` = index of ``(|i|, |j|)`` in A(d) and
  ``par[v] = ([i<0]|i| + [j<0]|j|) mod 2`` (diamond.py:63-71).

Lexicographic order on a centrally symmetric point set is reversed by
``p -> -p``: vertex ``v``'s antipode is ``nv - 1 - v``.  The device layout
(csrc/tcg.cu, build_layout) builds on that to turn the antipodal map into a swap of
mask halves.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ParseError
from .lattice import Point, index_of, num_points


def diamond_points(d: int) -> list[Point]:
    return [(i, j) for i in range(-d, d + 1) for j in range(-(d - abs(i)), d - abs(i) + 1)]


@dataclass(frozen=True)
class DiamondComplex:
    degree: int
    points: tuple[Point, ...]
    edges: tuple[tuple[int, int], ...]
    triangles: tuple[tuple[int, int, int], ...]
    antipodal_pairs: tuple[tuple[int, int], ...]

    def used_vertices(self) -> np.ndarray:
        used = np.zeros(len(self.points), dtype=np.uint8)
        for u, v in self.edges:
            used[u] = 1
            used[v] = 1
        return used

    @property
    def index(self) -> dict[Point, int]:
        return {p: k for k, p in enumerate(self.points)}

    def sign_extension_tables(self) -> tuple[np.ndarray, np.ndarray]:
        d = self.degree
        src = np.empty(len(self.points), dtype=np.int32)
        par = np.empty(len(self.points), dtype=np.uint8)
        for k, (i, j) in enumerate(self.points):
            src[k] = index_of(d, abs(i), abs(j))
            par[k] = ((-i if i < 0 else 0) + (-j if j < 0 else 0)) & 1
        return src, par


def reflect(T) -> DiamondComplex:
    d = int(T.degree)
    pts = diamond_points(d)
    idx = {p: k for k, p in enumerate(pts)}
    edges = set()
    tris = set()
    for sx in (1, -1):
        for sy in (1, -1):
            for p, q in T.edges:
                u = idx[(sx * int(p[0]), sy * int(p[1]))]
                v = idx[(sx * int(q[0]), sy * int(q[1]))]
                if u != v:
                    edges.add((u, v) if u < v else (v, u))
            for t in getattr(T, "triangles", ()):
                tris.add(tuple(sorted(idx[(sx * p[0], sy * p[1])] for p in t)))
    used = {u for e in edges for u in e}
    pairs = []
    for k, (i, j) in enumerate(pts):
        if abs(i) + abs(j) == d and (i, j) > (-i, -j) and k in used:
            pairs.append((idx[(-i, -j)], k))
    return DiamondComplex(d, tuple(pts), tuple(sorted(edges)), tuple(sorted(tris)), tuple(sorted(pairs)))


def extend_signs(D: DiamondComplex, sigma) -> np.ndarray:
    if sigma.degree != D.degree:
        raise ParseError(f"sign degree {sigma.degree} != diamond degree {D.degree}")
    src, par = D.sign_extension_tables()
    return np.asarray(sigma.bits, dtype=np.uint8)[src] ^ par


@dataclass(frozen=True)
class PlanArrays:
    """The reference plan tuple (classify.py:47-49) as flat arrays.

    This is exactly what the C ABI's ``tcg_desc`` points at.
    """

    degree: int
    nv: int
    npts: int
    edge_u: np.ndarray  # int32[ne]
    edge_v: np.ndarray  # int32[ne]
    src: np.ndarray  # int32[nv]
    par: np.ndarray  # uint8[nv]
    used: np.ndarray  # uint8[nv]
    ap_u: np.ndarray  # int32[2d]
    ap_v: np.ndarray  # int32[2d]
    maxreg: int


def plan_arrays(D: DiamondComplex) -> PlanArrays:
    from .lattice import harnack_bound

    d = D.degree
    src, par = D.sign_extension_tables()
    return PlanArrays(
        degree=d,
        nv=len(D.points),
        npts=num_points(d),
        edge_u=np.ascontiguousarray([e[0] for e in D.edges], dtype=np.int32),
        edge_v=np.ascontiguousarray([e[1] for e in D.edges], dtype=np.int32),
        src=np.ascontiguousarray(src, dtype=np.int32),
        par=np.ascontiguousarray(par, dtype=np.uint8),
        used=np.ascontiguousarray(D.used_vertices(), dtype=np.uint8),
        ap_u=np.ascontiguousarray([p[0] for p in D.antipodal_pairs], dtype=np.int32),
        ap_v=np.ascontiguousarray([p[1] for p in D.antipodal_pairs], dtype=np.int32),
        maxreg=harnack_bound(d) + 2,
    )
