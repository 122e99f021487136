"""How the sweep rate depends on the triangulation.

C3-style sweeps of 2^34 indices (one dedup window) for:
  * delaunay-7 (the staircase, the headline T) and the 16 random regular
    unimodular degree-7 triangulations c4-7-0..15 (reference generator,
    Random(0xB7)), raw [0, 2^34);
  * the degree-8 builtins (delaunay-8, bowtie8, fig2-middle8, fig2-right8),
    representative [2^38, 2^38 + 2^34).
Per T: patchworks/s (CUDA events around the sweep, after one warm-up sweep
of the same range), the tile / level-2 dedup counts and the explicit-
classification factor.  One JSON line per T; results/generalise_<tag>.json.

    python scripts/generalise.py [tag]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

from conftest import tri_from_fixture, triangulations  # noqa: E402
from paper_2604_09221_b200 import Classifier, builtin  # noqa: E402


def measure(name, T, raw, a, n):
    c = Classifier(T, device=0)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    c.native.set_stream(st.cuda_stream)
    c.native.agg_reset()
    c.native.sweep_async(raw, a, a + n)
    c.native.agg_fetch()
    c.native.tile_stats()
    c.native.level2_stats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c.native.agg_reset()
    e0.record(st)
    c.native.sweep_async(raw, a, a + n)
    e1.record(st)
    rc, bad, agg = c.native.agg_fetch()
    assert rc == 0, (name, rc, bad)
    ms = e0.elapsed_time(e1)
    tb, tc = c.native.tile_stats()
    l2b, l2c, l1 = c.native.level2_stats()
    bits = c.native.info["tile_bits_raw" if raw else "tile_bits_rep"]
    explicit = (l2c << 5) + (l1 << bits) if l2b else (tc << bits if tc else n)
    hist, total, keys, counts, wits = agg.result()
    return {"name": name, "degree": T.degree, "domain": "raw" if raw else "rep",
            "start": a, "n": n, "ms": ms, "patchworks_per_s": n / (ms / 1e3),
            "tiles": tb, "distinct_tiles": tc, "level2_records": l2b,
            "level2_distinct": l2c, "explicit_factor": n / explicit if explicit else None,
            "distinct_schemes": len(keys)}


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r2"
    tri = triangulations()
    jobs = [("delaunay-7", builtin("delaunay-7"), True, 0, 1 << 34)]
    jobs += [(f"c4-7-{k}", tri_from_fixture(tri[f"c4-7-{k}"]), True, 0, 1 << 34)
             for k in range(16)]
    jobs += [(nm, builtin(nm), False, 1 << 38, 1 << 34)
             for nm in ("delaunay-8", "bowtie8", "fig2-middle8", "fig2-right8")]
    out = []
    for job in jobs:
        r = measure(*job)
        print(json.dumps(r), flush=True)
        out.append(r)
    os.makedirs(os.path.join(ROOT, "results"), exist_ok=True)
    with open(os.path.join(ROOT, "results", f"generalise_{tag}.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
