"""Throughput of every BASELINE.json config on one GPU (device-timed with the
library's CUDA-event kernel timing; e2e = wall clock of the public call).

C1 d=4 raw 2^15 (tiny, correctness config) | C2 d=6 raw 2^28 | C3 d=7 raw 2^35
slice | C4 d=7 batch of random T x random signs | C5 d=8 sampling slices.
Prints one JSON object per config.
"""

from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2604_09221_b200 import Classifier, SweepRange, builtin, sample, sweep  # noqa: E402
from paper_2604_09221_b200.sweep import sample_slice  # noqa: E402


def timed(c, fn):
    c.native.kernel_times()
    c.native.set_timing(True)
    t0 = time.perf_counter()
    out = fn()
    wall = time.perf_counter() - t0
    c.native.set_timing(False)
    kt = c.native.kernel_times()
    dev = sum(v[0] for v in kt.values()) / 1e3
    return out, wall, dev, kt


def line(name, n, wall, dev, kt, extra=None):
    d = {"config": name, "patchworks": n, "device_s": round(dev, 4), "wall_s": round(wall, 4),
         "pps_device": n / dev if dev else None, "pps_e2e": n / wall,
         "kernels_ms": {k: round(v[0], 2) for k, v in kt.items() if v[1]}}
    if extra:
        d.update(extra)
    print(json.dumps(d), flush=True)


def main():
    which = sys.argv[1:] or ["C1", "C2", "C3", "C5", "C5sweep", "C4"]
    if "C1" in which:
        T = builtin("delaunay-4")
        c = Classifier(T)
        sweep(T, raw_space=True, classifier=c)
        r, wall, dev, kt = timed(c, lambda: sweep(T, raw_space=True, classifier=c))
        line("C1 delaunay-4 raw 2^15", 1 << 15, wall, dev, kt, {"hist": list(r.oval_histogram)})
    if "C2" in which:
        T = builtin("delaunay-6")
        c = Classifier(T)
        sweep(T, SweepRange(0, 1 << 24), raw_space=True, classifier=c)
        r, wall, dev, kt = timed(c, lambda: sweep(T, raw_space=True, classifier=c))
        line("C2 delaunay-6 raw 2^28 (full)", 1 << 28, wall, dev, kt,
             {"distinct": r.distinct_schemes(), "tiles": c.native.info["tile_bits_raw"]})
    if "C3" in which:
        T = builtin("delaunay-7")
        c = Classifier(T)
        a = 0x5A5A5A5A0 & ~((1 << 32) - 1)
        sweep(T, SweepRange(a, a + (1 << 26)), raw_space=True, classifier=c)
        r, wall, dev, kt = timed(c, lambda: sweep(T, SweepRange(a, a + (1 << 32)), raw_space=True,
                                                   classifier=c))
        line("C3 delaunay-7 raw 2^32 slice", 1 << 32, wall, dev, kt)
    if "C5" in which:
        for name in ("bowtie8", "delaunay-8"):
            T = builtin(name)
            c = Classifier(T)
            sample_slice(T, 20260810, 0, 1 << 22, classifier=c)
            n = 1 << 28
            r, wall, dev, kt = timed(c, lambda: sample_slice(T, 20260810, 1 << 39, (1 << 39) + n,
                                                              classifier=c))
            line(f"C5 {name} sample 2^28 draws at k0=2^39", n, wall, dev, kt,
                 {"hist_top": list(r.oval_histogram)})
    if "C5sweep" in which:
        for name in ("bowtie8", "delaunay-8"):
            T = builtin(name)
            c = Classifier(T)
            a = 1 << 38
            sweep(T, SweepRange(a, a + (1 << 24)), classifier=c)
            n = 1 << 30
            r, wall, dev, kt = timed(c, lambda: sweep(T, SweepRange(a, a + n), classifier=c))
            line(f"d=8 {name} rep sweep 2^30 at 2^38", n, wall, dev, kt,
                 {"tiles": c.native.info["tile_bits_rep"]})
    if "C4" in which:
        import random

        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from conftest import tri_from_fixture, triangulations

        tri = triangulations()
        Ts = [tri_from_fixture(tri[f"c4-7-{k}"]) for k in range(16)]
        cs = [Classifier(T) for T in Ts]
        rng = np.random.default_rng(7)
        n = 1 << 22
        words = rng.integers(0, 1 << 36, size=n, dtype=np.uint64)
        for c in cs:
            c.classify_words(words[:1024])
        tot_dev = tot_wall = 0.0
        for c in cs:
            _, wall, dev, kt = timed(c, lambda c=c: c.classify_words(words))
            tot_dev += dev
            tot_wall += wall
        line("C4 16 random d=7 T x 2^22 random signs (per-T batches)", 16 * n, tot_wall, tot_dev,
             {"batch": (tot_dev * 1e3, 16)})
        random.seed(0)


if __name__ == "__main__":
    main()
