"""GPU parity: the CUDA path (through the C ABI) against the reference's own
outputs (tests/golden/, produced by the reference) and the CPU oracle."""

import numpy as np
import pytest

from conftest import golden, plan_dict, tri_from_fixture, triangulations

pytestmark = pytest.mark.gpu


def _classifier(t):
    from paper_2604_09221_b200 import Classifier

    return Classifier(tri_from_fixture(t), device=0)


def test_pairs_match_reference():
    from paper_2604_09221_b200.scheme import scheme_from_key

    tri = triangulations()
    n = 0
    for e in golden("pairs.json"):
        t = tri[e["name"]]
        c = _classifier(t)
        words = np.array([int(s[::-1], 2) for s, *_ in e["rows"]], np.uint64)
        keys, ov, nr, st = c.classify_words(words)
        for i, (s, scheme, ovals, nreg) in enumerate(e["rows"]):
            assert st[i] == 0, (e["name"], s, st[i])
            assert scheme_from_key(int(keys[i]), t["degree"] % 2 == 1) == scheme, (e["name"], s)
            assert (int(ov[i]), int(nr[i])) == (ovals, nreg)
            n += 1
    assert n > 2500


def test_garbage_statuses_match_reference():
    from paper_2604_09221_b200 import _lib
    from paper_2604_09221_b200.diamond import PlanArrays
    from paper_2604_09221_b200.scheme import scheme_from_key

    for e in golden("garbage.json"):
        P = plan_dict(e)
        arr = PlanArrays(P["degree"], P["nv"], P["npts"], np.array(P["edge_u"], np.int32),
                         np.array(P["edge_v"], np.int32), np.array(P["src"], np.int32),
                         np.array(P["par"], np.uint8), np.array(P["used"], np.uint8),
                         np.array(P["ap_u"], np.int32), np.array(P["ap_v"], np.int32),
                         P["maxreg"])
        plan = _lib.NativePlan(arr, 0)
        words = np.array([r[0] for r in e["rows"]], np.uint64)
        keys, ov, nr, st = plan.classify_words(words)
        for i, (m, status, ovals, nreg, scheme) in enumerate(e["rows"]):
            assert int(st[i]) == status, (e["name"], m, int(st[i]), status)
            if status == 0:
                assert scheme_from_key(int(keys[i]), e["degree"] % 2 == 1) == scheme
                assert (int(ov[i]), int(nr[i])) == (ovals, nreg)


def _check_report(rep, g):
    from paper_2604_09221_b200.io import histogram_csv, report_jsonl

    assert list(rep.oval_histogram) == g["hist"]
    assert rep.total_classified == g["total"]
    assert rep.scheme_map == {s: tuple(v) for s, v in g["schemes"].items()}
    assert rep.fingerprint == g["fingerprint"]
    assert histogram_csv(rep) == g["csv"]
    if g["params"].get("mode") in ("sweep", "sample"):
        assert report_jsonl(rep) == g["jsonl"]


def test_reports_match_reference():
    from paper_2604_09221_b200 import SweepRange, builtin, sample, sweep
    from paper_2604_09221_b200.lattice import validate_triangulation

    for name, g in golden("reports.json").items():
        parts = name.split("-")
        if "edges" in g:
            edges = [((a, b), (c, e)) for a, b, c, e in g["edges"]]
            T = validate_triangulation(g["degree"], edges, require_unimodular=False)
        elif parts[1] in ("delaunay",):
            T = builtin(f"delaunay-{parts[2]}")
        else:
            T = builtin(parts[1] if parts[1] != "fig2" else f"fig2-{parts[2]}")
        p = g["params"]
        if p["mode"] == "sweep":
            rep = sweep(T, SweepRange(p["start"], p["end"]), raw_space=p["raw_space"])
        else:
            rep = sample(T, p["n"], p["seed"])
        _check_report(rep, g)


def test_c2_full_rep_sweep_delaunay6():
    from paper_2604_09221_b200 import builtin, sweep

    g = golden("c2_delaunay6_rep.json")
    _check_report(sweep(builtin("delaunay-6")), g)


def test_c3_slices_delaunay7():
    from paper_2604_09221_b200 import SweepRange, builtin, sweep, Classifier

    T = builtin("delaunay-7")
    c = Classifier(T, device=0)
    for s in golden("c3_delaunay7_raw_slices.json")["slices"]:
        rep = sweep(T, SweepRange(s["start"], s["end"]), raw_space=True, classifier=c)
        assert list(rep.oval_histogram) == s["hist"]
        assert rep.scheme_map == {k: tuple(v) for k, v in s["schemes"].items()}


def test_c5_sample_slices_degree8():
    from paper_2604_09221_b200 import builtin, Classifier
    from paper_2604_09221_b200.sweep import sample_slice

    cache = {}
    for s in golden("c5_sample_slices.json")["slices"]:
        T = builtin(s["name"])
        c = cache.setdefault(s["name"], Classifier(T, device=0))
        rep = sample_slice(T, s["seed"], s["k0"], s["k1"], classifier=c)
        assert list(rep.oval_histogram) == s["hist"], (s["name"], s["k0"])
        assert rep.scheme_map == {k: tuple(v) for k, v in s["schemes"].items()}


def test_generic_engine_matches_reference_every_degree():
    """The any-degree kernel (one CTA per patchwork) on every pair fixture:
    d = 1..9 (pairs.json) and d = 10..48 (pairs_large.json)."""
    from paper_2604_09221_b200 import Classifier
    from paper_2604_09221_b200.lattice import validate_triangulation

    tri = triangulations()
    for e in golden("pairs.json"):
        c = Classifier(tri_from_fixture(tri[e["name"]]), device=0, engine="generic")
        res = c.classify_many([s for s, *_ in e["rows"]])
        for (s, scheme, ov, nr), r in zip(e["rows"], res):
            assert (r.scheme, r.oval_count, r.region_count) == (scheme, ov, nr), (e["name"], s)
    for e in golden("pairs_large.json"):
        edges = [((a, b), (c2, f)) for a, b, c2, f in e["edges"]]
        c = Classifier(validate_triangulation(e["degree"], edges), device=0)
        assert c.generic
        res = c.classify_many([s for s, *_ in e["rows"]])
        for (s, scheme, ov, nr), r in zip(e["rows"], res):
            assert (r.scheme, r.oval_count, r.region_count) == (scheme, ov, nr), (e["name"], s)


def test_generic_engine_statuses_match_reference():
    from paper_2604_09221_b200 import _lib
    from paper_2604_09221_b200.diamond import PlanArrays

    for e in golden("garbage.json"):
        P = plan_dict(e)
        arr = PlanArrays(P["degree"], P["nv"], P["npts"], np.array(P["edge_u"], np.int32),
                         np.array(P["edge_v"], np.int32), np.array(P["src"], np.int32),
                         np.array(P["par"], np.uint8), np.array(P["used"], np.uint8),
                         np.array(P["ap_u"], np.int32), np.array(P["ap_v"], np.int32),
                         P["maxreg"])
        g = _lib.NativeLarge(arr, 0)
        rows = np.array([[r[0]] for r in e["rows"]], np.uint64)
        st, nr, par = g.classify_rows(rows)
        for i, (m, status, ovals, nreg, scheme) in enumerate(e["rows"]):
            assert int(st[i]) == status, (e["name"], m, int(st[i]), status)
            if status == 0:
                assert (int(nr[i]) - 1, int(nr[i])) == (ovals, nreg)


def test_acceptance_criterion_10_degree_scaling():
    """time(d=48) / time(d=24) <= 5 through _run_bits (test_acceptance.py:223-253)."""
    import random as _random
    import time

    from paper_2604_09221_b200 import Classifier, lattice_points, num_points
    from paper_2604_09221_b200.lifting import from_lifting

    rng = _random.Random(0x5CA1E)

    def mean_call(d, calls):
        T = None
        while T is None or not T.is_unimodular:  # exact lifting: redraw degenerate jitter
            lift = {(i, j): 8 * (i * i + i * j + j * j) + rng.randint(0, 1)
                    for i, j in lattice_points(d)}
            T = from_lifting(d, lift)
        c = Classifier(T, device=0)
        batches = [np.array([rng.randint(0, 1) for _ in range(num_points(d))], np.uint8)
                   for _ in range(calls)]
        for b in batches[:10]:
            c._run_bits(b)
        best = float("inf")
        for _ in range(5):
            t0 = time.perf_counter()
            for b in batches:
                c._run_bits(b)
            best = min(best, (time.perf_counter() - t0) / calls)
        return best

    t24, t48 = mean_call(24, 60), mean_call(48, 30)
    assert t48 / t24 <= 5.0, (t24, t48)


@pytest.mark.gpu
def test_large_kernel_deterministic_under_repetition():
    """k_large (any degree) gives the same status and tree on every repetition:
    a halving find in its flatten phase once left a stale ancestor in the
    union-find and, rarely, reported NOT_A_TREE (1 in ~2,400 calls at d=24)."""
    import random as _random

    from paper_2604_09221_b200 import Classifier, lattice_points, num_points
    from paper_2604_09221_b200.lifting import from_lifting

    rng = _random.Random(0x5CA1E)
    d = 24
    T = None
    while T is None or not T.is_unimodular:
        lift = {(i, j): 8 * (i * i + i * j + j * j) + rng.randint(0, 1) for i, j in lattice_points(d)}
        T = from_lifting(d, lift)
    c = Classifier(T, device=0)
    words = (num_points(d) + 63) // 64
    gen = np.random.default_rng(24)
    rows = gen.integers(0, 2**63, size=(256, words), dtype=np.uint64)
    rows[:, -1] &= np.uint64((1 << (num_points(d) - 64 * (words - 1))) - 1)
    st0, nr0, par0 = c.large.classify_rows(rows)
    for _ in range(40):
        st, nr, par = c.large.classify_rows(rows)
        assert np.array_equal(st, st0) and np.array_equal(nr, nr0)
        for t in range(len(rows)):
            if st0[t] == 0:
                assert np.array_equal(par[t][: nr0[t]], par0[t][: nr0[t]])
