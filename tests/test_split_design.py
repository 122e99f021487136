"""Host-side separator design of the split sampler (csrc/split_design.cuh),
run through the C ABI without a GPU (tcg_split_design).

The sampler is exact only if the separator F really separates: no edge of T
may join a point of side A to a point of side B (then the same-sign
components of each side depend on that side's signs alone), and antipodal
links, which join copies of one lattice point, stay inside a side.  The
table index bits are the sides' free (non-pinned) points.
"""

import pytest

from conftest import tri_from_fixture, triangulations

NAMES = ["bowtie8", "delaunay-8", "fig2-middle8", "fig2-right8", "delaunay-9", "delaunay-7",
         "delaunay-6", "random-8-0", "random-8-1", "random-7-2", "c4-7-5", "random-6-0"]


def _tri(name):
    from paper_2604_09221_b200 import builtin

    t = triangulations().get(name)
    return tri_from_fixture(t) if t is not None else builtin(name)


@pytest.mark.parametrize("name", NAMES)
def test_separator_splits_the_point_graph(name):
    from paper_2604_09221_b200 import _lib
    from paper_2604_09221_b200.diamond import plan_arrays, reflect
    from paper_2604_09221_b200.lattice import index_of, num_points

    T = _tri(name)
    d = T.degree
    arr = plan_arrays(reflect(T))
    des = _lib.split_design(arr)
    assert des is not None, name
    F, A, B = des["F"], des["A"], des["B"]
    npts = num_points(d)
    assert F & A == 0 and F & B == 0 and A & B == 0
    assert F | A | B == (1 << npts) - 1
    assert A and B and F
    for p, q in T.edges:
        a, b = index_of(d, *p), index_of(d, *q)
        assert not ((A >> a) & 1 and (B >> b) & 1), (p, q)
        assert not ((B >> a) & 1 and (A >> b) & 1), (p, q)
    pinned = (1 << 0) | (1 << 1) | (1 << (d + 1))
    assert des["bits_a"] == bin(A & ~pinned).count("1")
    assert des["bits_b"] == bin(B & ~pinned).count("1")
    assert max(des["bits_a"], des["bits_b"]) <= 24
    nF = sum(1 for v in range(arr.nv) if arr.used[v] and (F >> int(arr.src[v])) & 1)
    assert des["separator_vertices"] == nF <= 32
    assert 0 < des["mean_nodes"] <= 64
    assert des["table_bytes"] <= 4 << 30


def test_design_is_deterministic():
    from paper_2604_09221_b200 import _lib, builtin
    from paper_2604_09221_b200.diamond import plan_arrays, reflect

    arr = plan_arrays(reflect(builtin("bowtie8")))
    assert _lib.split_design(arr) == _lib.split_design(arr)


def test_low_degrees_have_no_split():
    from paper_2604_09221_b200 import _lib, builtin
    from paper_2604_09221_b200.diamond import plan_arrays, reflect

    # the design itself exists for any degree; the plan only uses it for d >= 6
    des = _lib.split_design(plan_arrays(reflect(builtin("delaunay-3"))))
    assert des is None or des["separator_vertices"] >= 1
