"""Pin the CPU oracle (oracle/tcg_oracle.c) to the reference's own outputs.

The oracle is only trusted as a checker because these tests hold it
bit-exact to fixtures the reference produced (tests/golden/make_golden.py).
"""

import numpy as np
import pytest

from conftest import golden, plan_dict, tri_from_fixture, triangulations

from oracle import oracle as O
from paper_2604_09221_b200 import builtin
from paper_2604_09221_b200.diamond import plan_arrays, reflect


def _oplan(T):
    return O.OraclePlan.from_arrays(plan_arrays(reflect(T)))


def test_oracle_pairs_match_reference():
    tri = triangulations()
    n = 0
    for e in golden("pairs.json"):
        plan = O.OraclePlan.from_arrays(plan_dict(tri[e["name"]]))
        words = [int(s[::-1], 2) for s, *_ in e["rows"]]
        for (s, scheme, ov, nr), got in zip(e["rows"], O.classify_words(plan, words)):
            assert got == (0, scheme, ov, nr), (e["name"], s)
            n += 1
    assert n > 2500


def test_oracle_statuses_match_reference():
    seen = set()
    for e in golden("garbage.json"):
        plan = O.OraclePlan.from_arrays(plan_dict(e))
        got = O.classify_words(plan, [r[0] for r in e["rows"]])
        for (m, status, ov, nr, scheme), (st, sch, o, n) in zip(e["rows"], got):
            assert st == status, (e["name"], m)
            seen.add(st)
            if st == 0:
                assert (sch, o, n) == (scheme, ov, nr)
    assert {0, 2, 3, 7} <= seen


@pytest.mark.parametrize("name", ["sweep-delaunay-4-raw", "sweep-delaunay-5-rep",
                                  "sweep-delaunay-3-40-100", "sweep-spike-3-raw",
                                  "sweep-random-5-rep", "sweep-delaunay-7-raw-0-65536"])
def test_oracle_sweeps_match_reference(name):
    g = golden("reports.json")[name]
    if "edges" in g:
        T = tri_from_fixture({"degree": g["degree"], "edges": g["edges"], "unimodular": None})
    else:
        T = builtin(f"delaunay-{g['degree']}")
    p = g["params"]
    r = O.sweep(_oplan(T), p["raw_space"], p["start"], p["end"], threads=4)
    assert r["status"] == 0
    assert r["hist"][: len(g["hist"])] == g["hist"]
    assert r["schemes"] == {s: tuple(v) for s, v in g["schemes"].items()}
    assert r["total"] == g["total"]


def test_oracle_c1_goldens():
    # d=4 raw histogram and witnesses
    r = O.sweep(_oplan(builtin("delaunay-4")), True, 0, 1 << 15, threads=4)
    assert r["hist"][:5] == [0, 14336, 14336, 3584, 512]
    assert r["schemes"] == {"<1<1>>": (3584, 0), "<1>": (14336, 2), "<2>": (10752, 4),
                            "<3>": (3584, 72), "<4>": (512, 1034)}


def test_oracle_samples_match_reference():
    g = golden("reports.json")
    for name in ("sample-delaunay-4-5000-42", "sample-bowtie8-50000-20260810",
                 "sample-delaunay-9-20000-9"):
        e = g[name]
        T = builtin(name.split("-")[1] if "bowtie" in name else f"delaunay-{e['degree']}")
        nbits = (e["degree"] + 1) * (e["degree"] + 2) // 2 - 3
        r = O.sample(_oplan(T), e["params"]["seed"], 0, e["params"]["n"], nbits, threads=4)
        assert r["hist"][: len(e["hist"])] == e["hist"]
        assert r["schemes"] == {s: tuple(v) for s, v in e["schemes"].items()}


def test_oracle_c3_and_c5_slices():
    """Two of the sixteen C3 slices and two C5 sample slices (2^20 each)."""
    T7 = builtin("delaunay-7")
    p7 = _oplan(T7)
    for s in golden("c3_delaunay7_raw_slices.json")["slices"][:2]:
        r = O.sweep(p7, True, s["start"], s["end"], threads=8)
        assert r["hist"][: len(s["hist"])] == s["hist"]
        assert r["schemes"] == {k: tuple(v) for k, v in s["schemes"].items()}
    for s in golden("c5_sample_slices.json")["slices"][::6][:2]:
        r = O.sample(_oplan(builtin(s["name"])), s["seed"], s["k0"], s["k1"], 42, threads=8)
        assert r["hist"][: len(s["hist"])] == s["hist"]
        assert r["schemes"] == {k: tuple(v) for k, v in s["schemes"].items()}


def test_splitmix64_known_values():
    # kernels.py:439-444 on the reference's own constants
    z = (20260810 + 1 * 0x9E3779B97F4A7C15) % 2**64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) % 2**64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) % 2**64
    assert O.splitmix64(20260810, 0) == z ^ (z >> 31)


def test_oracle_worker_invariance():
    p = _oplan(builtin("delaunay-5"))
    a = O.sweep(p, False, 0, 1 << 18, threads=1)
    b = O.sweep(p, False, 0, 1 << 18, threads=8, chunk=977)
    assert a == b
    assert np.sum(a["hist"]) == 1 << 18


def test_oracle_large_degrees_match_reference():
    """d = 10..48 (beyond the 64-bit sign word), fixtures from the reference."""
    from paper_2604_09221_b200.lattice import validate_triangulation

    for e in golden("pairs_large.json"):
        edges = [((a, b), (c, f)) for a, b, c, f in e["edges"]]
        T = validate_triangulation(e["degree"], edges)
        assert T.fingerprint() == e["fingerprint"]
        got = O.classify_bitstrings(_oplan(T), [r[0] for r in e["rows"]])
        for (s, scheme, ov, nr), g in zip(e["rows"], got):
            assert g == (0, scheme, ov, nr), (e["name"], s)


def test_oracle_every_status_matches_reference():
    """Statuses 1-8 on bad plans (tests/golden/status.json, kernels.py:183-266)."""
    seen = set()
    for e in golden("status.json"):
        P = plan_dict(e)
        got = O.classify_words(O.OraclePlan.from_arrays(P), [r[0] for r in e["rows"]])
        for (m, status, *_), (st, *_r) in zip(e["rows"], got):
            assert st == status, (e["name"], m)
            seen.add(st)
    assert seen == {1, 2, 3, 4, 5, 6, 7, 8}


def test_oracle_differential_criterion():
    """test_acceptance.py:144-160 replayed: 25 T x 10^4 signs per degree 1..6."""
    from conftest import diff_triangulation

    for g in golden("diff.json"):
        d = g["degree"]
        plans = [_oplan(diff_triangulation(d, e)) for e in g["triangulations"]]
        rows = np.array(g["rows"], dtype=np.int64)
        for k, plan in enumerate(plans):
            sel = rows[rows[:, 0] == k]
            got = O.classify_words(plan, sel[:, 1].astype(np.uint64))
            for r, (st, s, ov, nr) in zip(sel, got):
                assert (st, s, ov, nr) == (0, g["schemes"][r[2]], r[3], r[4]), (d, k, r[1])


def test_oracle_garbage_sweeps_first_failure():
    """sweep_kernel's (status, smallest failing index) on rare-failure plans."""
    import os

    for e in golden("garbage_sweep.json"):
        r = O.sweep(O.OraclePlan.from_arrays(plan_dict(e)), e["raw"], e["start"], e["end"],
                    threads=os.cpu_count() or 1)
        assert (r["status"], r["bad"]) == (e["status"], e["bad"]), e["name"]
