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
