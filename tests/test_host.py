"""CPU tests of the host side: preprocessing, codecs, canonical strings, tree
keys and report writers, pinned to fixtures the reference produced."""

import random

import pytest
from hypothesis import given, settings, strategies as st

from conftest import golden, tri_from_fixture, triangulations

from paper_2604_09221_b200 import (
    IndexOutOfRange,
    MergeMismatch,
    NotATriangulation,
    NotUnimodular,
    ParseError,
    PointOutOfRange,
    SignDistribution,
    builtin,
    empty_report,
    merge,
    normalize_sign,
    num_representatives,
    representative,
)
from paper_2604_09221_b200.diamond import plan_arrays, reflect
from paper_2604_09221_b200.io import histogram_csv, report_jsonl
from paper_2604_09221_b200.lattice import validate_triangulation
from paper_2604_09221_b200.scheme import (
    SchemeNode,
    SchemeTree,
    canonical_scheme,
    key_from_tree,
    key_ovals,
    parse_scheme,
    scheme_from_key,
    tree_from_key,
)
from paper_2604_09221_b200.signs import (
    eps_action,
    raw_index,
    rep_to_sigma,
    sigma_to_rep,
    sign_from_raw_index,
)
from paper_2604_09221_b200.sweep import SweepReport


# ------------------------------------------------------------ preprocessing
def test_plans_match_reference_plans():
    """reflect + sign tables + antipodal pairs == the reference's plan tuple."""
    for name, t in triangulations().items():
        T = tri_from_fixture(t)
        assert T.fingerprint() == t["fingerprint"], name
        P = plan_arrays(reflect(T))
        g = t["plan"]
        for k in ("edge_u", "edge_v", "src", "par", "used", "ap_u", "ap_v"):
            assert getattr(P, k).tolist() == g[k], (name, k)
        assert (P.nv, P.npts, P.maxreg) == (g["nv"], g["npts"], g["maxreg"])


def test_builtins_match_reference_edges():
    tri = triangulations()
    for d in range(1, 10):
        T = builtin(f"delaunay-{d}")
        assert [list(p) + list(q) for p, q in T.edges] == tri[f"delaunay-{d}"]["edges"]
        assert T.is_unimodular
    for name in ("bowtie8", "fig2-middle8", "fig2-right8"):
        T = builtin(name)
        assert T.fingerprint() == tri[name]["fingerprint"]
        assert T.is_unimodular


def test_reflection_counts():
    # test_acceptance.py:107-111
    expected = {2: 28, 3: 60, 4: 104, 5: 160, 6: 228, 7: 308, 8: 400}
    for d, n in expected.items():
        assert len(reflect(builtin(f"delaunay-{d}")).edges) == n


def test_validation_errors():
    with pytest.raises(PointOutOfRange):
        validate_triangulation(2, [((0, 0), (3, 0))])
    with pytest.raises(NotATriangulation):
        validate_triangulation(2, [((0, 0), (0, 0))])
    with pytest.raises(NotATriangulation):
        validate_triangulation(1, [((0, 0), (1, 0))])
    with pytest.raises(NotATriangulation):  # crossing diagonals
        validate_triangulation(2, list(builtin("delaunay-2").edges) + [((0, 0), (1, 1))])
    spike = triangulations()["spike-3"]
    edges = [((a, b), (c, e)) for a, b, c, e in spike["edges"]]
    with pytest.raises(NotUnimodular):
        validate_triangulation(3, edges)
    assert not validate_triangulation(3, edges, require_unimodular=False).is_unimodular


# ------------------------------------------------------------------ codecs
def test_representative_examples():
    # test_sweep.py:25-30
    assert representative(2, 0).bitstring() == "000000"
    assert representative(2, 1).bitstring() == "001000"
    assert num_representatives(2) == 8
    assert num_representatives(1) == 1
    with pytest.raises(IndexOutOfRange):
        representative(2, 8)


@given(st.integers(0, num_representatives(4) - 1))
@settings(max_examples=200, deadline=None)
def test_representative_roundtrip(m):
    rep, back = normalize_sign(representative(4, m))
    assert back == m and rep == representative(4, m)
    assert sigma_to_rep(4, rep_to_sigma(4, m)) == m


def test_normalize_lands_in_orbit(rng):
    for d in (2, 3, 4, 7):
        n = (d + 1) * (d + 2) // 2
        for _ in range(20):
            s = SignDistribution.from_bitstring(d, "".join(rng.choice("01") for _ in range(n)))
            rep, m = normalize_sign(s)
            assert rep.bits[0] == rep.bits[1] == rep.bits[d + 1] == 0
            orbit = {eps_action(s, (a, b, c)).bitstring()
                     for a in (0, 1) for b in (0, 1) for c in (0, 1)}
            assert rep.bitstring() in orbit
            assert sign_from_raw_index(d, raw_index(s)) == s


def test_bitstring_errors():
    with pytest.raises(ParseError):
        SignDistribution.from_bitstring(2, "000")
    with pytest.raises(ParseError):
        SignDistribution.from_bitstring(1, "01x")


# ------------------------------------------------------- canonical strings
KATS = ["<0>", "<J>", "<3>", "<J u 1<1>>", "<2 u 1<2>>", "<2<1>>", "<1<1> u 1<2>>",
        "<9 u 1<1>>", "<J u 15>", "<18 u 1<3>>", "<1 u 1<5>>", "<1<1<1>>>"]


def test_scheme_kats_roundtrip():
    for s in KATS:
        t = parse_scheme(s)
        assert canonical_scheme(t) == s
        assert scheme_from_key(key_from_tree(t.root), t.has_pseudoline) == s


def _trees(depth=4):
    return st.recursive(st.just(SchemeNode()),
                        lambda kids: st.lists(kids, max_size=4).map(SchemeNode),
                        max_leaves=25)


@given(_trees(), st.booleans())
@settings(max_examples=300, deadline=None)
def test_tree_key_is_canonical(root, odd):
    """The AHU key is an isomorphism invariant and decodes to the reference string."""
    k = key_from_tree(root)
    tree = SchemeTree(root, odd)
    assert scheme_from_key(k, odd) == canonical_scheme(tree)
    assert key_ovals(k) == tree.oval_count()
    # shuffling children does not change the key
    rnd = random.Random(k & 0xFFFF)

    def shuffled(n):
        kids = [shuffled(c) for c in n.children]
        rnd.shuffle(kids)
        return SchemeNode(kids)

    assert key_from_tree(shuffled(root)) == k
    assert key_from_tree(tree_from_key(k)) == k


def test_parse_errors():
    for bad in ("<", "<J u J>", "<0 u 1>", "<1<>", "<1> ", "<x>"):
        with pytest.raises(ParseError):
            parse_scheme(bad)


# ----------------------------------------------------------------- reports
def _report(g):
    return SweepReport(g["degree"], g["fingerprint"], g["raw_space"], tuple(g["hist"]),
                       {s: tuple(v) for s, v in g["schemes"].items()}, g["total"], g["params"])


def test_report_writers_byte_identical():
    """report_jsonl / histogram_csv reproduce the reference's files byte for byte."""
    for name, g in golden("reports.json").items():
        r = _report(g)
        assert histogram_csv(r) == g["csv"], name
        assert report_jsonl(r) == g["jsonl"], name


def test_merge_properties_on_reference_reports():
    g = golden("reports.json")
    a = _report(g["sweep-delaunay-3-0-40"])
    b = _report(g["sweep-delaunay-3-40-100"])
    c = _report(g["sweep-delaunay-3-100-128"])
    full = _report(g["sweep-delaunay-3-rep"])
    assert merge(merge(a, b), c) == full
    assert merge(a, merge(b, c)) == full
    assert merge(a, b) == merge(b, a)
    assert merge(a, empty_report(builtin("delaunay-3"))) == a
    with pytest.raises(MergeMismatch):
        merge(a, _report(g["sweep-delaunay-3-raw"]))
