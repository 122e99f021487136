"""Regular triangulations from liftings (host side; config C4 workloads).

A lifting assigns an integer height to every point of A(d); the lower convex
hull of the lifted points projects to a regular subdivision (the reference's
lifting.py:1-141 uses symbolic perturbation to always return a
triangulation).  Here qhull proposes the lower facets and every facet is
then certified with exact integer arithmetic (all other lifted points
strictly above its plane); a lifting with any degenerate facet is rejected
instead of perturbed, so accepted liftings give exactly the regular
triangulation they induce.  ``random_unimodular`` draws from the same
family as the reference's test fixture (convex quadratic base plus bounded
jitter, tests/conftest.py:8-25), rejecting until unimodular.
"""

from __future__ import annotations

import numpy as np

from .errors import InvalidDegree, NotATriangulation
from .lattice import Triangulation, lattice_points, validate_triangulation


def delaunay_lifting(d: int) -> dict:
    return {(i, j): i * i + i * j + j * j for i, j in lattice_points(d)}


def random_lifting(d: int, rng, base: int = 4) -> dict:
    a, c = rng.randint(1, 3), rng.randint(1, 3)
    b = rng.randint(0, min(a, c))
    return {(i, j): base * (a * i * i + b * i * j + c * j * j) + rng.randint(0, 2 * base)
            for i, j in lattice_points(d)}


def _above(p, q, r, s) -> int:
    """Sign of the lifted s over the plane through lifted p, q, r ((x, y, h) ints),
    oriented so that a counterclockwise (p, q, r) gives +1 for 'strictly above'."""
    ax, ay, ah = q[0] - p[0], q[1] - p[1], q[2] - p[2]
    bx, by, bh = r[0] - p[0], r[1] - p[1], r[2] - p[2]
    cx, cy, ch = s[0] - p[0], s[1] - p[1], s[2] - p[2]
    det = ax * (by * ch - bh * cy) - ay * (bx * ch - bh * cx) + ah * (bx * cy - by * cx)
    orient = ax * by - ay * bx
    return (det > 0) - (det < 0) if orient > 0 else -((det > 0) - (det < 0))


def from_lifting(d: int, lifting: dict) -> Triangulation | None:
    """The regular triangulation induced by a generic lifting, or None if some
    lower facet is not a certified triangle (degenerate lifting)."""
    if d < 1:
        raise InvalidDegree(f"degree must be >= 1, got {d}")
    from scipy.spatial import ConvexHull

    pts = lattice_points(d)
    P = np.array([(i, j, int(lifting[(i, j)])) for i, j in pts], dtype=np.float64)
    hull = ConvexHull(P)
    lower = [s for s, eq in zip(hull.simplices, hull.equations) if eq[2] < -1e-12]
    lifted = [(i, j, int(lifting[(i, j)])) for i, j in pts]
    edges = set()
    for tri in lower:
        a, b, c = (int(x) for x in tri)
        pa, pb, pc = lifted[a], lifted[b], lifted[c]
        if (pb[0] - pa[0]) * (pc[1] - pa[1]) - (pb[1] - pa[1]) * (pc[0] - pa[0]) == 0:
            continue  # vertical facet over a boundary segment
        for k in range(len(pts)):
            if k in (a, b, c):
                continue
            if _above(pa, pb, pc, lifted[k]) <= 0:
                return None
        for u, v in ((a, b), (b, c), (a, c)):
            p, q = pts[u], pts[v]
            edges.add((p, q) if p <= q else (q, p))
    try:
        return validate_triangulation(d, sorted(edges), require_unimodular=False)
    except NotATriangulation:
        return None


def random_unimodular(d: int, rng, max_tries: int = 2000) -> Triangulation:
    for _ in range(max_tries):
        T = from_lifting(d, random_lifting(d, rng))
        if T is not None and T.is_unimodular:
            return T
    raise AssertionError(f"could not draw a unimodular degree-{d} triangulation")
