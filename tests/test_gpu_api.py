"""GPU tests of the drop-in API, mirroring the reference's own test suite
(test_classify.py, test_sweep.py, test_acceptance.py) plus full-size
property checks the oracle cannot reach in seconds."""

import itertools
import random

import numpy as np
import pytest

from conftest import golden, plan_dict, tri_from_fixture, triangulations

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    import paper_2604_09221_b200 as api

    return api


def _bits(d, rng):
    return "".join(rng.choice("01") for _ in range((d + 1) * (d + 2) // 2))


def test_degree1_all_eight(api):
    c = api.Classifier(api.builtin("delaunay-1"))
    for bits in itertools.product("01", repeat=3):
        assert c.classify("".join(bits)).scheme == "<J>"
    rep = api.sweep(api.builtin("delaunay-1"), raw_space=True, classifier=c)
    assert rep.total_classified == 8 and set(rep.scheme_map) == {"<J>"}
    assert api.sweep(api.builtin("delaunay-1")).scheme_map == {"<J>": (1, 0)}


def test_degree2_sweeps(api):
    T = api.builtin("delaunay-2")
    rep = api.sweep(T)
    assert rep.total_classified == 8 and set(rep.scheme_map) == {"<1>"}
    raw = api.sweep(T, raw_space=True)
    assert raw.total_classified == 64 and raw.max_ovals() == 1
    assert raw.witness_bitstring("<1>") == "000000"
    assert api.classify(T, "000000").scheme == "<1>"


def test_invariances(api, rng):
    """(Z/2)^3 sign action and the S3 symmetry (test_classify.py:68-89)."""
    for name in ("random-3-0", "random-4-1", "random-5-2", "delaunay-7", "bowtie8"):
        T = tri_from_fixture(triangulations()[name])
        d = T.degree
        c = api.Classifier(T)
        for _ in range(10):
            s = api.SignDistribution.from_bitstring(d, _bits(d, rng))
            base = c.classify(s)
            many = c.classify_many([api.eps_action(s, e)
                                    for e in itertools.product((0, 1), repeat=3)])
            assert all(r == base for r in many)
        for g in api.SYMMETRY_GROUP:
            gT, _ = api.apply_symmetry(T, None, g)
            cg = api.Classifier(gT)
            for _ in range(5):
                s = api.SignDistribution.from_bitstring(d, _bits(d, rng))
                _, gs = api.apply_symmetry(T, s, g)
                assert cg.classify(gs) == c.classify(s)


def test_structural_invariants(api, rng):
    # test_acceptance.py:188-201
    for d in range(1, 10):
        c = api.Classifier(api.builtin(f"delaunay-{d}"))
        res = c.classify_many([_bits(d, rng) for _ in range(300)])
        for r in res:
            assert r.region_count == r.oval_count + 1
            assert r.oval_count + (d % 2) <= api.harnack_bound(d)
            assert r.has_pseudoline == (d % 2 == 1)
            assert ("J" in r.scheme) == (d % 2 == 1)


def test_bowtie_even_ovals(api, rng):
    c = api.Classifier(api.builtin("bowtie8"))
    for r in c.classify_many([_bits(8, rng) for _ in range(2000)]):
        assert r.oval_count % 2 == 0 and r.oval_count >= 4


def test_harnack_m_curves(api):
    # sigma(i,j) = i*j mod 2 on delaunay-d
    want = {4: "<4>", 5: "<J u 6>", 6: "<9 u 1<1>>", 7: "<J u 15>", 8: "<18 u 1<3>>"}
    for d, s in want.items():
        c = api.Classifier(api.builtin(f"delaunay-{d}"))
        bits = "".join(str((i * j) % 2) for i, j in api.lattice_points(d))
        r = c.classify(bits)
        assert r.scheme == s and r.oval_count == api.harnack_bound(d) - (d % 2)


def test_chunk_split_merge_and_witness_minimality(api):
    T = api.builtin("delaunay-3")
    full = api.sweep(T)
    k = api.num_representatives(3) // 2
    assert api.merge(api.sweep(T, api.SweepRange(0, k)),
                     api.sweep(T, api.SweepRange(k, 2 * k))) == full
    c = api.Classifier(T)
    for scheme, (count, wit) in full.scheme_map.items():
        assert c.classify(api.representative(3, wit)).scheme == scheme
        others = c.classify_many([api.representative(3, m) for m in range(wit)])
        assert all(r.scheme != scheme for r in others)


def test_full_size_split_invariance_degree7(api):
    """2^32 raw indices as one launch chain == split at an odd point and merged."""
    T = api.builtin("delaunay-7")
    c = api.Classifier(T)
    a, b, m = 5 << 30, (5 << 30) + (1 << 32), (5 << 30) + 1234567891
    whole = api.sweep(T, api.SweepRange(a, b), raw_space=True, classifier=c)
    parts = api.merge(api.sweep(T, api.SweepRange(a, m), raw_space=True, classifier=c),
                      api.sweep(T, api.SweepRange(m, b), raw_space=True, classifier=c))
    assert whole == parts
    assert whole.total_classified == 1 << 32 == sum(whole.oval_histogram)
    assert sum(c for c, _ in whole.scheme_map.values()) == 1 << 32


def test_raw_vs_rep_domain_relations(api):
    """raw counts = 8 x rep counts; raw lower half = raw / 2 with equal witnesses
    (verified there for d = 3, 4, 5)."""
    for d in (4, 5, 6):
        T = api.builtin(f"delaunay-{d}")
        c = api.Classifier(T)
        n = (d + 1) * (d + 2) // 2
        rep = api.sweep(T, classifier=c)
        raw = api.sweep(T, raw_space=True, classifier=c)
        low = api.sweep(T, api.SweepRange(0, 1 << (n - 1)), raw_space=True, classifier=c)
        assert set(rep.scheme_map) == set(raw.scheme_map) == set(low.scheme_map)
        for s, (cnt, w) in raw.scheme_map.items():
            assert cnt == 8 * rep.scheme_map[s][0]
            assert low.scheme_map[s] == (cnt // 2, w)


def test_sample_reproducible_and_partition_independent(api):
    T = api.builtin("delaunay-4")
    c = api.Classifier(T)
    a = api.sample(T, 5000, seed=42, classifier=c)
    assert a == api.sample(T, 5000, seed=42, workers=4, chunk_size=977, classifier=c)
    assert a.total_classified == 5000
    assert api.sample(T, 5000, seed=43, classifier=c) != a
    T8 = api.builtin("bowtie8")
    c8 = api.Classifier(T8)
    full = api.sample(T8, 300_000, seed=5, classifier=c8)
    from paper_2604_09221_b200.sweep import sample_slice

    s1 = sample_slice(T8, 5, 0, 123_457, classifier=c8)
    s2 = sample_slice(T8, 5, 123_457, 300_000, classifier=c8)
    merged = api.merge(s1, s2)
    assert merged.oval_histogram == full.oval_histogram
    assert merged.scheme_map == full.scheme_map


def test_fig2_bowtie_distribution(api):
    # test_acceptance.py:128-141 (criterion 05), +-0.3 pp on 10^6 draws
    bins = {4: 4.6875, 6: 11.3281, 8: 14.6484, 10: 25.5371, 12: 17.1997, 14: 13.9526,
            16: 10.9695, 18: 1.6113, 20: 0.0652, 22: 0.0004}
    r = api.sample(api.builtin("bowtie8"), 1_000_000, seed=20260810)
    assert r.total_classified == 1_000_000
    for k, c in enumerate(r.oval_histogram):
        if k % 2 == 1 or k < 4:
            assert c == 0
    for k, pct in bins.items():
        assert abs(100.0 * r.oval_histogram[k] / 1_000_000 - pct) <= 0.3
    assert "<0>" not in r.scheme_map and r.distinct_schemes() <= 123


def test_errors(api):
    T = api.builtin("delaunay-2")
    with pytest.raises(api.IndexOutOfRange):
        api.sweep(T, api.SweepRange(0, 9))
    with pytest.raises(api.IndexOutOfRange):
        api.SweepRange(5, 3)
    with pytest.raises(api.BudgetExceeded):
        api.sweep(api.builtin("delaunay-10"))
    with pytest.raises(api.ParseError):
        api.Classifier(T).classify("000")
    with pytest.raises(api.IndexOutOfRange):
        api.sample(T, 0, seed=1)


def test_sweep_error_reports_smallest_failing_index(api):
    """A garbage plan fails inside the sweep kernel; the raised index and
    message are those of the oracle's first failing index."""
    from oracle import oracle as O
    from paper_2604_09221_b200 import _lib
    from paper_2604_09221_b200.classify import STATUS_MESSAGES
    from paper_2604_09221_b200.diamond import PlanArrays
    from paper_2604_09221_b200.sweep import _raise_status

    e = [g for g in golden("garbage.json") if g["name"] == "garbage-5-0"][0]
    P = plan_dict(e)
    arr = PlanArrays(P["degree"], P["nv"], P["npts"], np.array(P["edge_u"], np.int32),
                     np.array(P["edge_v"], np.int32), np.array(P["src"], np.int32),
                     np.array(P["par"], np.uint8), np.array(P["used"], np.uint8),
                     np.array(P["ap_u"], np.int32), np.array(P["ap_v"], np.int32), P["maxreg"])
    plan = _lib.NativePlan(arr, 0)
    rc, bad, _ = plan.sweep(True, 1000, 1000 + (1 << 16))
    ref = O.sweep(O.OraclePlan.from_arrays(P), True, 1000, 1000 + (1 << 16), threads=1)
    assert ref["status"] != 0
    assert (rc, bad) == (ref["status"], ref["bad"])
    with pytest.raises(api.InvariantViolation, match=STATUS_MESSAGES[rc]):
        _raise_status(rc, bad)


def test_c4_random_triangulations_batch(api):
    """Config C4: random regular unimodular degree-7 T x random signs, per pair."""
    from oracle import oracle as O

    tri = triangulations()
    rng = np.random.default_rng(0xB7)
    for k in range(16):
        t = tri[f"c4-7-{k}"]
        c = api.Classifier(tri_from_fixture(t))
        words = rng.integers(0, 1 << 36, size=2048, dtype=np.uint64)
        keys, ov, nr, st = c.classify_words(words)
        ref = O.classify_words(O.OraclePlan.from_arrays(plan_dict(t)), words)
        for i, (s, scheme, o, n) in enumerate(ref):
            assert st[i] == s == 0
            assert api.scheme_from_key(int(keys[i]), True) == scheme
            assert (int(ov[i]), int(nr[i])) == (o, n)


def test_multi_device_api_single_device(api):
    T = api.builtin("delaunay-5")
    a = api.sweep(T, devices=[0])
    assert a == api.sweep(T)


def test_multi_plan_sweeps_and_samples_equal_single_plan(api):
    """tcg_sweep_multi / tcg_sample_multi with two and three distinct plans on
    device 0 (one host thread each) == one plan; plans are cached per entry."""
    T = api.builtin("delaunay-7")
    c = api.Classifier(T)
    a, b = 3 << 30, (3 << 30) + (1 << 28) + 12345
    single = api.sweep(T, api.SweepRange(a, b), raw_space=True, classifier=c)
    for devs in ([0, 0], [0, 0, 0]):
        multi = api.sweep(T, api.SweepRange(a, b), raw_space=True, classifier=c, devices=devs)
        assert multi == single
    plans = c.device_plans([0, 0, 0])
    assert len({id(p) for p in plans}) == 3 and plans[0] is c.native
    assert all(x is y for x, y in zip(plans, c.device_plans([0, 0, 0])))
    T8 = api.builtin("bowtie8")
    c8 = api.Classifier(T8)
    s1 = api.sample(T8, 400_000, seed=5, classifier=c8)
    s2 = api.sample(T8, 400_000, seed=5, classifier=c8, devices=[0, 0])
    assert s1 == s2


def test_multi_rejects_a_plan_listed_twice(api):
    from paper_2604_09221_b200 import _lib

    c = api.Classifier(api.builtin("delaunay-5"))
    with pytest.raises(api.DeviceError, match="listed twice"):
        _lib.sweep_multi([c.native, c.native], True, 0, 1 << 20)


def test_multi_plan_failure_is_the_earliest(api):
    """A failing plan sharded over 3 plans reports the same (status, index) as
    one plan: the earliest failure in index order, whichever shard holds it."""
    from paper_2604_09221_b200 import _lib

    from conftest import plan_arrays_of

    e = golden("garbage_sweep.json")[0]
    arr = plan_arrays_of(plan_dict(e))
    plans = [_lib.NativePlan(arr, 0) for _ in range(3)]
    rc, bad, _ = _lib.sweep_multi(plans, e["raw"], e["start"], e["end"])
    assert (rc, bad) == (e["status"], e["bad"])


def test_report_bytes_identical_across_call_shapes(api):
    # criterion 09: byte-identical reports for any partition
    from paper_2604_09221_b200.io import histogram_csv, report_jsonl

    for d in (2, 3, 4, 5):
        T = api.builtin(f"delaunay-{d}")
        c = api.Classifier(T)
        outs = {report_jsonl(api.sweep(T, workers=w, chunk_size=cs, classifier=c))
                + histogram_csv(api.sweep(T, classifier=c))
                for w, cs in ((1, 65536), (2, 111), (8, 4096))}
        assert len(outs) == 1


def test_multi_triangulation_batch_matches_oracle(api):
    """Config C4 through MultiClassifier: one launch, one topology per CTA."""
    import random as _random

    from oracle import oracle as O
    from paper_2604_09221_b200.diamond import plan_arrays, reflect
    from paper_2604_09221_b200.lifting import random_unimodular

    rng = _random.Random(0xB7)
    Ts = [random_unimodular(7, rng) for _ in range(48)]
    Ts += [tri_from_fixture(triangulations()[f"c4-7-{k}"]) for k in range(16)]
    mc = api.MultiClassifier(Ts)
    g = np.random.default_rng(4)
    n = 1 << 16
    tri = g.integers(0, len(Ts), size=n).astype(np.int32)
    words = g.integers(0, 1 << 36, size=n, dtype=np.uint64)
    keys, ov, nr, st = mc.classify_words(tri, words)
    assert (st == 0).all()
    for t in range(len(Ts)):
        sel = np.nonzero(tri == t)[0][:64]
        ref = O.classify_words(O.OraclePlan.from_arrays(plan_arrays(reflect(Ts[t]))), words[sel])
        for i, (s, scheme, o, r) in zip(sel, ref):
            assert api.scheme_from_key(int(keys[i]), True) == scheme
            assert (int(ov[i]), int(nr[i])) == (o, r)
    pairs = [(int(tri[i]), "".join(str((int(words[i]) >> k) & 1) for k in range(36)))
             for i in range(200)]
    res = mc.classify_pairs(pairs)
    assert [r.scheme for r in res] == [api.scheme_from_key(int(keys[i]), True)
                                       for i in range(200)]


def test_cli_reports_byte_identical_to_reference(api, tmp_path, capsys):
    from paper_2604_09221_b200.cli import main

    g = golden("reports.json")["sweep-delaunay-4-raw"]
    out, hist = tmp_path / "r.jsonl", tmp_path / "h.csv"
    code = main(["sweep", "--builtin", "delaunay-4", "--raw-sign-space", "--output", str(out),
                 "--histogram", str(hist)])
    assert code == 0
    assert out.read_text() == g["jsonl"] and hist.read_text() == g["csv"]
    code = main(["classify", "--builtin", "delaunay-2", "000000", "--json"])
    assert code == 0
    assert '"scheme": "<1>"' in capsys.readouterr().out
    s = golden("reports.json")["sample-delaunay-4-5000-42"]
    code = main(["sample", "--builtin", "delaunay-4", "-n", "5000", "--seed", "42",
                 "--output", str(out), "--histogram", str(hist)])
    assert code == 0 and out.read_text() == s["jsonl"] and hist.read_text() == s["csv"]


def test_large_batch_pipeline_consistent(api):
    """Batches larger than one pinned staging chunk (2^20) equal small batches."""
    c = api.Classifier(api.builtin("delaunay-7"))
    g = np.random.default_rng(11)
    n = 3 * (1 << 20) + 12345
    words = g.integers(0, 1 << 36, size=n, dtype=np.uint64)
    keys, ov, nr, st = c.classify_words(words)
    assert (st == 0).all()
    for lo in (0, (1 << 20) - 7, 2 * (1 << 20) + 999, n - 5000):
        k2, o2, r2, s2 = c.classify_words(words[lo:lo + 5000])
        assert (k2 == keys[lo:lo + 5000]).all() and (o2 == ov[lo:lo + 5000]).all()
        assert (r2 == nr[lo:lo + 5000]).all() and (s2 == 0).all()


def test_tile_fallback_path_is_exact():
    """Force every tile through the full-diamond fallback (contraction limit
    lowered in a subprocess) and compare with the contracted path."""
    import json
    import os
    import subprocess
    import sys

    code = (
        "import json,sys; sys.path.insert(0, %r)\n"
        "from paper_2604_09221_b200 import builtin, sweep, SweepRange\n"
        "out = {}\n"
        "for name, raw, a in (('delaunay-7', True, 12345678), ('delaunay-6', False, 777),"
        " ('bowtie8', False, 1 << 38)):\n"
        "    r = sweep(builtin(name), SweepRange(a, a + (1 << 18) + 77), raw_space=raw)\n"
        "    out[name] = [list(r.oval_histogram), sorted(r.scheme_map.items())]\n"
        "print(json.dumps(out))\n" % os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    res = {}
    for limit in ("64", "8"):
        env = dict(os.environ, TCG_TILE_MAXNODES=limit)
        p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        assert p.returncode == 0, p.stderr
        res[limit] = json.loads(p.stdout.strip().splitlines()[-1])
    assert res["64"] == res["8"]


def test_two_rank_sharded_sweep_equals_single_process():
    """distributed.sweep_sharded with 2 ranks (gloo collectives, both ranks on
    cuda:0) merges to exactly the single-process report."""
    import os
    import socket
    import subprocess
    import sys

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                        str(port), os.path.join(root, "scripts", "sharded_check.py")],
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    assert "sharded == single: True" in p.stdout


@pytest.mark.parametrize("name,raw,a,n", [
    ("delaunay-7", True, 0x5A5A5A5A0 + 3, (1 << 24) + 1001),
    ("delaunay-6", True, 12345, 1 << 24),
    ("delaunay-6", False, 0, 1 << 25),
    ("bowtie8", False, (1 << 38) + 17, 1 << 25),
    ("delaunay-8", False, 1 << 39, 1 << 24),
])
def test_tile_dedup_is_exact(api, name, raw, a, n):
    """Classifying each distinct contracted tile once, weighted by its
    multiplicity, gives the identical report (counts, histogram, witnesses)."""
    T = api.builtin(name)
    c = api.Classifier(T)
    reps = {}
    for on in (False, True):
        c.native.set_dedup(on)
        c.native.tile_stats()
        r = api.sweep(T, api.SweepRange(a, a + n), raw_space=raw, classifier=c)
        built, classified = c.native.tile_stats()
        reps[on] = (r.oval_histogram, sorted(r.scheme_map.items()), r.total_classified)
        if on:
            assert 0 < classified <= built
        else:
            assert classified == built  # every tile classified
    c.native.set_dedup(None)
    assert reps[True] == reps[False]


def test_tile_dedup_chunk_size_invariance():
    """Small contraction chunks (fewer duplicates per chunk) give the same report."""
    import json
    import os
    import subprocess
    import sys

    code = (
        "import json,sys; sys.path.insert(0, %r)\n"
        "from paper_2604_09221_b200 import builtin, sweep, SweepRange\n"
        "r = sweep(builtin('delaunay-7'), SweepRange(99, 99 + (1 << 25)), raw_space=True)\n"
        "print(json.dumps([list(r.oval_histogram), sorted(r.scheme_map.items())]))\n"
        % os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    res = {}
    for lg in ("14", "21"):
        env = dict(os.environ, TCG_CHUNK_LOG2=lg)
        p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        assert p.returncode == 0, p.stderr
        res[lg] = json.loads(p.stdout.strip().splitlines()[-1])
    assert res["14"] == res["21"]


@pytest.mark.parametrize("name,raw,a,n", [
    ("delaunay-7", True, 0x5A5A5A5A0 + 3, (1 << 24) + 1001),
    ("delaunay-7", False, 777, 1 << 24),
    ("delaunay-5", True, 0, 1 << 21),
    ("delaunay-7", True, 0, 1 << 26),
    ("delaunay-6", True, 12345, 1 << 24),
    ("delaunay-6", False, 0, 1 << 25),
    ("bowtie8", False, (1 << 38) + 17, 1 << 25),
    ("delaunay-8", False, 1 << 39, 1 << 24),
    ("fig2-middle8", False, 3 << 38, 1 << 24),
    ("fig2-right8", False, 5 << 37, 1 << 24),
])
def test_level2_contraction_is_exact(api, name, raw, a, n):
    """Level-2 records (A points fixed, super-nodes) deduplicated and
    classified per lane give the identical report as the level-1 path."""
    T = api.builtin(name)
    c = api.Classifier(T)
    reps = {}
    for on in (False, True):
        c.native.set_level2(on)
        c.native.level2_stats()
        r = api.sweep(T, api.SweepRange(a, a + n), raw_space=raw, classifier=c)
        built, classified, _ = c.native.level2_stats()
        reps[on] = (r.oval_histogram, sorted(r.scheme_map.items()), r.total_classified)
        if on and T.degree in (6, 7):
            assert 0 < classified < built
        if not on:
            assert built == 0
    c.native.set_level2(None)
    assert reps[True] == reps[False]


def test_super_tile_records_identical_to_direct_contraction():
    """Tiles contracted from their super-tile's record (TCG_SUPER_BITS 4 and 6)
    are byte-identical to the direct contraction (TCG_BUILD_GENERIC=1): the
    deduplication finds exactly the same number of distinct tiles, and the
    reports are equal."""
    import json
    import os
    import subprocess
    import sys

    code = (
        "import json,sys; sys.path.insert(0, %r)\n"
        "import random\n"
        "from paper_2604_09221_b200 import builtin, sweep, SweepRange, Classifier\n"
        "from paper_2604_09221_b200.lifting import random_unimodular\n"
        "out = []\n"
        "cases = [(builtin('delaunay-7'), True, 0x5A5A5A5A0 + 3, (1 << 24) + 1001),\n"
        "         (builtin('delaunay-6'), False, 777, 1 << 22),\n"
        "         (builtin('delaunay-5'), True, 5, 1 << 20),\n"
        "         (builtin('bowtie8'), False, (1 << 38) + 17, 1 << 23),\n"
        "         (builtin('delaunay-8'), False, 1 << 39, 1 << 22),\n"
        "         (random_unimodular(7, random.Random(0xB7)), True, 1 << 33, 1 << 22)]\n"
        "for T, raw, a, n in cases:\n"
        "    c = Classifier(T)\n"
        "    c.native.tile_stats()\n"
        "    r = sweep(T, SweepRange(a, a + n), raw_space=raw, classifier=c)\n"
        "    out.append([list(r.oval_histogram), sorted(r.scheme_map.items()),\n"
        "                list(c.native.tile_stats())])\n"
        "print(json.dumps(out))\n" % os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    res = {}
    for tag, extra in (("generic", {"TCG_BUILD_GENERIC": "1"}), ("super4", {"TCG_SUPER_BITS": "4"}),
                       ("super6", {"TCG_SUPER_BITS": "6"})):
        env = dict(os.environ, **extra)
        p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        assert p.returncode == 0, p.stderr
        res[tag] = json.loads(p.stdout.strip().splitlines()[-1])
    assert res["super4"] == res["generic"]
    assert res["super6"] == res["generic"]


def test_two_stage_level2_identical_to_direct():
    """Two-stage level-2 records (A1 bits fixed, deduplicated, then A2) give
    the same reports as building level-2 records directly (TCG_L2_TWOSTAGE=0),
    also when a small stage-1 budget sends batches back to the direct build."""
    import json
    import os
    import subprocess
    import sys

    code = (
        "import json,sys; sys.path.insert(0, %r)\n"
        "import random\n"
        "from paper_2604_09221_b200 import builtin, sweep, SweepRange\n"
        "from paper_2604_09221_b200.lifting import random_unimodular\n"
        "out = []\n"
        "for T, raw, a, n in [(builtin('delaunay-7'), True, 0x5A5A5A5A0 + 3, (1 << 25) + 1001),\n"
        "                     (builtin('delaunay-7'), True, 0, 1 << 26),\n"
        "                     (builtin('delaunay-7'), False, 777, 1 << 24),\n"
        "                     (random_unimodular(7, random.Random(0xB7)), True, 1 << 33, 1 << 24)]:\n"
        "    r = sweep(T, SweepRange(a, a + n), raw_space=raw)\n"
        "    out.append([list(r.oval_histogram), sorted(r.scheme_map.items())])\n"
        "print(json.dumps(out))\n" % os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    res = {}
    for flag, extra in (("0", {}), ("1", {}), ("1", {"TCG_L15_MAXM": "6"})):
        env = dict(os.environ, TCG_L2_TWOSTAGE=flag, **extra)
        p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        assert p.returncode == 0, p.stderr
        res[flag + "".join(extra)] = json.loads(p.stdout.strip().splitlines()[-1])
    # the third run forces stage-1 budget overflows: batches go back to the direct build
    assert res["0"] == res["1"] == res["1TCG_L15_MAXM"]


def test_pipeline_deterministic_across_grid_shapes():
    """Race canary (compute-sanitizer is unavailable on this GPU pool): the
    d=7 and d=8 sweep pipelines give byte-identical reports whatever the
    grid shapes of the two-stage kernels (CTAs per SM of the stage-1 build,
    its dedup, stage 2, the direct level-2 build), run twice each."""
    import json
    import os
    import subprocess
    import sys

    code = (
        "import json,sys; sys.path.insert(0, %r)\n"
        "from paper_2604_09221_b200 import builtin, sweep, SweepRange\n"
        "from paper_2604_09221_b200.io import report_jsonl\n"
        "out = []\n"
        "for name, raw, a, n in (('delaunay-7', True, 0x5A5A5A5A0 + 3, (1 << 27) + 1001),\n"
        "                        ('bowtie8', False, (1 << 38) + 17, 1 << 26)):\n"
        "    for rep in range(2):\n"
        "        out.append(report_jsonl(sweep(builtin(name), SweepRange(a, a + n), raw_space=raw)))\n"
        "print(json.dumps(out))\n" % os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    res = []
    for env in ({}, {"TCG_L15_GRID": "3", "TCG_L15D_GRID": "2", "TCG_L2F_GRID": "8",
                     "TCG_L2B_GRID": "1"},
                {"TCG_L15_GRID": "1", "TCG_L15D_GRID": "32", "TCG_L2F_GRID": "1",
                 "TCG_L2B_GRID": "32"}):
        p = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env),
                           capture_output=True, text=True)
        assert p.returncode == 0, p.stderr[-2000:]
        res.append(json.loads(p.stdout.strip().splitlines()[-1]))
    for r in res:
        assert r[0] == r[1] == res[0][0] and r[2] == r[3] == res[0][2]


_MULTI_CHUNKED = r'''
import sys, numpy as np
sys.path.insert(0, ".")
from paper_2604_09221_b200 import Classifier, MultiClassifier
from paper_2604_09221_b200.lifting import random_unimodular
import random
rng = random.Random(0xC4)
Ts = [random_unimodular(7, rng) for _ in range(24)]
mc = MultiClassifier(Ts, device=0)
g = np.random.default_rng(9)
n = (1 << 20) + 12345
words = g.integers(0, 1 << 36, size=n, dtype=np.uint64)
tri_sorted = np.sort(g.integers(0, len(Ts), size=n)).astype(np.int32)   # grouped: no regrouping
tri_random = g.permutation(tri_sorted).astype(np.int32)                 # regrouped + scattered
for tri in (tri_sorted, tri_random):
    keys, ov, nr, st = mc.classify_words(tri, words)
    assert (st == 0).all()
    for t in range(len(Ts)):
        sel = np.nonzero(tri == t)[0]
        k1, o1, r1, s1 = Classifier(Ts[t], device=0).classify_words(words[sel])
        assert (keys[sel] == k1).all() and (ov[sel] == o1).all() and (nr[sel] == r1).all()
print("ok")
'''


def test_multi_triangulation_pipeline_chunks(api, tmp_path):
    """tcg_multi_classify's pinned-staging pipeline over many chunks (2^18
    pairs each, ~4 per call), grouped and regrouped inputs, against the
    single-triangulation batch path."""
    import os
    import subprocess
    import sys

    script = tmp_path / "chunked.py"
    script.write_text(_MULTI_CHUNKED)
    env = dict(os.environ, TCG_MULTI_CHUNK_LOG2="18")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, str(script)], cwd=root, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]
