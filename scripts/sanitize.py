"""compute-sanitizer target: one small launch chain of one kernel family.

    compute-sanitizer --tool racecheck python scripts/sanitize.py <family>

Families (kernels exercised):
  batch     k_batch<K,EVEN> (d = 4, 7, 8: K = 2, 4, 6)
  enum      k_enumerate raw / rep / sample (d = 4 raw sweep, d = 8 sample)
  sweep7    d = 7 raw sweep through the pipeline: k_super_build,
            k_tile_from_super, k_tile_dedup, k_l15_build, k_l2_dedup,
            k_l2_from_l15, k_l2_classify, k_tile_classify (range ends),
            k_agg_clear, k_agg_compact
  direct7   same with TCG_L2_TWOSTAGE=0: k_l2_build<false>
  sweep8    d = 8 representative sweep (even degree): k_l2_build<true>,
            k_l2_classify_even, k_tile_build_lanes fallback tiles
  sweep6    d = 6 raw sweep (even, K = 4 tiles)
  multi     k_multi (many triangulations)
  large     k_large (d = 10, any-degree engine)
  split     k_split_build, k_sample_split, k_sample_list (d = 8 sampling through
            the separator-split tables, forced fallbacks)
Each run checks its result against the reference fixtures it can reach
(tests/golden), so a sanitizer pass also shows the launch computed the
right answer under instrumentation.
"""
import json
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

fam = sys.argv[1]
if fam == "direct7":
    os.environ["TCG_L2_TWOSTAGE"] = "0"

from paper_2604_09221_b200 import (  # noqa: E402
    Classifier, MultiClassifier, SweepRange, builtin, sweep)
from paper_2604_09221_b200.sweep import sample_slice  # noqa: E402


def golden(name):
    with open(os.path.join(ROOT, "tests", "golden", name)) as fh:
        return json.load(fh)


def check(rep, g):
    assert list(rep.oval_histogram) == g["hist"][:len(rep.oval_histogram)], "hist"
    assert rep.scheme_map == {k: tuple(v) for k, v in g["schemes"].items()}, "schemes"


if fam == "batch":
    pairs = {e["name"]: e["rows"] for e in golden("pairs.json")}
    for name in ("delaunay-4", "delaunay-7", "bowtie8"):
        c = Classifier(builtin(name))
        rows = pairs[name]
        res = c.classify_many([r[0] for r in rows])
        assert [r.scheme for r in res] == [r[1] for r in rows], name
elif fam == "enum":
    g = golden("reports.json")
    check(sweep(builtin("delaunay-4"), raw_space=True), g["sweep-delaunay-4-raw"])
    s = [x for x in golden("c5_sample_slices.json")["slices"] if x["name"] == "bowtie8"][0]
    T = builtin("bowtie8")
    r = sample_slice(T, s["seed"], s["k0"], s["k0"] + (1 << 14))
    assert r.total_classified == 1 << 14
elif fam in ("sweep7", "direct7"):
    g = golden("c3_delaunay7_raw_slices.json")["slices"][0]
    check(sweep(builtin("delaunay-7"), SweepRange(g["start"], g["end"]), raw_space=True), g)
elif fam == "sweep8":
    T = builtin("bowtie8")
    a = (1 << 38) + 17
    r = sweep(T, SweepRange(a, a + (1 << 20)))
    assert r.total_classified == 1 << 20
elif fam == "sweep6":
    g = golden("c2_delaunay6_rep.json")
    r = sweep(builtin("delaunay-6"), SweepRange(0, 1 << 21))
    assert r.total_classified == 1 << 21 and set(r.scheme_map) <= set(g["schemes"])
elif fam == "split":
    os.environ["TCG_SPLIT_MAXNODES"] = "44"  # some draws take the flat list kernel
    for s in [x for x in golden("c5_sample_slices.json")["slices"] if x["k0"] == 0]:
        T = builtin(s["name"])
        c = Classifier(T)
        c.native.set_split(True)
        r = sample_slice(T, s["seed"], s["k0"], s["k1"], classifier=c)
        check(r, s)
        st = c.native.split_stats()
        assert st[0] == 1 and st[2] > 0, st
elif fam == "multi":
    from paper_2604_09221_b200.lifting import random_unimodular

    rng = random.Random(0xB7)
    Ts = [random_unimodular(7, rng) for _ in range(8)]
    mc = MultiClassifier(Ts)
    w = np.random.default_rng(1).integers(0, 1 << 36, size=4096, dtype=np.uint64)
    t = (np.arange(4096) % 8).astype(np.int32)
    keys, ov, nr, st = mc.classify_words(t, w)
    assert (st == 0).all()
elif fam == "large":
    big = [e for e in golden("pairs_large.json") if e["name"] == "delaunay-10"][0]
    c = Classifier(builtin("delaunay-10"))
    res = c.classify_many([r[0] for r in big["rows"][:8]])
    assert [r.scheme for r in res] == [r[1] for r in big["rows"][:8]]
else:
    raise SystemExit(f"unknown family {fam}")
print("sanitize target ok:", fam)
