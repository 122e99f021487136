"""Generate the golden fixtures under tests/golden/ from the reference package.

Test infrastructure only.  Run in the build container, where the reference
(`tcurves`, Python + numba) is importable from /root/reference/pkg/src:

    NUMBA_CACHE_DIR=/tmp/nbcache python tests/golden/make_golden.py [part ...]

Parts: tri, pairs, garbage, reports, c2, c3, c5, fig (default: all).
Every value written here is produced by the reference's own public API or
its compiled kernels (kernels.py:366, 423, 447); nothing is computed by
this repo's code.  The GPU box never runs this script: the JSON it writes
is committed and travels with the repo.
"""

from __future__ import annotations

import json
import os
import random
import sys
import time

REF = os.environ.get("TCURVES_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nbcache")

import numpy as np  # noqa: E402

import tcurves  # noqa: E402
from tcurves import (  # noqa: E402
    Classifier,
    SweepRange,
    builtin,
    from_lifting,
    lattice_points,
    sample,
    sweep,
)
from tcurves import kernels  # noqa: E402
import importlib  # noqa: E402

sweep_mod = importlib.import_module("tcurves.sweep")
from tcurves.io import histogram_csv, report_jsonl  # noqa: E402
from tcurves.lattice import Triangulation  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
WORKERS = os.cpu_count() or 1


# ---------------------------------------------------------------- generators
# Same distribution as the reference's tests/conftest.py:8-25 (convex
# quadratic lifting plus bounded jitter, rejection-sampled for unimodularity).
def random_lifting(d, rng, base=4):
    a, c = rng.randint(1, 3), rng.randint(1, 3)
    b = rng.randint(0, min(a, c))
    jitter = 2 * base
    return {
        (i, j): base * (a * i * i + b * i * j + c * j * j) + rng.randint(0, jitter)
        for i, j in lattice_points(d)
    }


def random_unimodular(d, rng, max_tries=2000):
    for _ in range(max_tries):
        T = from_lifting(d, random_lifting(d, rng))
        if T.is_unimodular:
            return T
    raise AssertionError(d)


def random_bits(d, rng):
    n = len(lattice_points(d))
    return "".join(rng.choice("01") for _ in range(n))


def edges_flat(T):
    return [[p[0], p[1], q[0], q[1]] for p, q in T.edges]


def plan_dict(c: Classifier):
    d, nv, npts, eu, ev, src, par, used, apu, apv, maxreg = c._plan_common
    return {
        "nv": int(nv),
        "npts": int(npts),
        "edge_u": eu.tolist(),
        "edge_v": ev.tolist(),
        "src": src.tolist(),
        "par": par.tolist(),
        "used": used.tolist(),
        "ap_u": apu.tolist(),
        "ap_v": apv.tolist(),
        "maxreg": int(maxreg),
    }


def report_dict(r):
    return {
        "degree": r.degree,
        "fingerprint": r.fingerprint,
        "raw_space": r.raw_space,
        "hist": list(r.oval_histogram),
        "schemes": {s: [c, w] for s, (c, w) in sorted(r.scheme_map.items())},
        "total": r.total_classified,
        "params": r.params,
        "jsonl": report_jsonl(r),
        "csv": histogram_csv(r),
    }


def dump(name, obj):
    path = os.path.join(OUT, name)
    with open(path, "w") as fh:
        json.dump(obj, fh, separators=(",", ":"), sort_keys=True)
        fh.write("\n")
    print(f"wrote {path} ({os.path.getsize(path)} bytes)", flush=True)


# ---------------------------------------------------------------- parts
def triangulation_pool():
    """Named triangulations used across fixtures (deterministic)."""
    pool = []
    for d in range(1, 10):
        pool.append((f"delaunay-{d}", builtin(f"delaunay-{d}")))
    for name in ("bowtie8", "fig2-middle8", "fig2-right8"):
        pool.append((name, builtin(name)))
    rng = random.Random(0xC0FFEE)
    for d in range(1, 9):
        for k in range(3):
            pool.append((f"random-{d}-{k}", random_unimodular(d, rng)))
    lift = {p: 0 for p in lattice_points(3)}
    lift[(1, 1)] = 7
    pool.append(("spike-3", from_lifting(3, lift)))  # non-unimodular (test_classify.py:54-65)
    lift = {p: 0 for p in lattice_points(5)}
    lift[(2, 1)] = 9
    lift[(1, 2)] = 9
    pool.append(("spike-5", from_lifting(5, lift)))
    rng = random.Random(0xB7)
    for k in range(16):
        pool.append((f"c4-7-{k}", random_unimodular(7, rng)))
    return pool


def part_tri():
    out = []
    for name, T in triangulation_pool():
        c = Classifier(T)
        out.append(
            {
                "name": name,
                "degree": T.degree,
                "edges": edges_flat(T),
                "fingerprint": T.fingerprint(),
                "unimodular": bool(T.is_unimodular),
                "plan": plan_dict(c),
            }
        )
    dump("triangulations.json", out)


def part_pairs():
    rng = random.Random(1234)
    out = []
    for name, T in triangulation_pool():
        c = Classifier(T)
        d = T.degree
        sigmas = [random_bits(d, rng) for _ in range(48)]
        if name.startswith("delaunay-"):
            # Harnack signs (i*j mod 2) and the all-plus / all-minus vectors
            sigmas.append("".join(str((i * j) % 2) for i, j in lattice_points(d)))
            sigmas.append("0" * len(lattice_points(d)))
            sigmas.append("1" * len(lattice_points(d)))
        rows = []
        for s in sigmas:
            r = c.classify(s)
            rows.append([s, r.scheme, r.oval_count, r.region_count])
        out.append({"name": name, "rows": rows})
    dump("pairs.json", out)


def part_garbage():
    """Statuses of the compiled kernel on non-triangulation edge sets.

    Triangulation objects are built directly (no validation), as an
    unvalidated caller could; classify_bits_kernel then reports the
    reference's status codes (kernels.py:20-45).
    """
    rng = random.Random(0x6A5B)
    out = []
    for d in (2, 3, 4, 5, 6, 7, 8):
        base = builtin(f"delaunay-{d}")
        pts = lattice_points(d)
        for variant in range(6):
            edges = list(base.edges)
            if variant % 3 == 0:  # drop edges
                k = max(1, len(edges) // (4 + variant))
                for _ in range(k):
                    edges.pop(rng.randrange(len(edges)))
            elif variant % 3 == 1:  # add random chords
                for _ in range(2 + variant):
                    p, q = rng.sample(pts, 2)
                    e = (p, q) if p < q else (q, p)
                    if e not in edges:
                        edges.append(e)
            else:  # both
                for _ in range(3):
                    edges.pop(rng.randrange(len(edges)))
                for _ in range(3):
                    p, q = rng.sample(pts, 2)
                    e = (p, q) if p < q else (q, p)
                    if e not in edges:
                        edges.append(e)
            T = Triangulation(d, tuple(sorted(edges)), ())
            c = Classifier(T)
            plan = c.plan(raw_space=True)
            scr = c.make_scratch()
            rows = []
            for _ in range(64):
                m = rng.getrandbits(len(pts))
                bits = np.array([(m >> k) & 1 for k in range(len(pts))], dtype=np.uint8)
                st, ov, nr, ln = kernels.classify_bits_kernel(plan, scr, bits)
                scheme = bytes(scr[27][:ln]).decode() if st == 0 else None
                rows.append([m, int(st), int(ov), int(nr), scheme])
            out.append(
                {
                    "name": f"garbage-{d}-{variant}",
                    "degree": d,
                    "edges": [[p[0], p[1], q[0], q[1]] for p, q in T.edges],
                    "plan": plan_dict(c),
                    "rows": rows,
                }
            )
    dump("garbage.json", out)


def part_reports():
    out = {}
    for d in range(1, 6):
        T = builtin(f"delaunay-{d}")
        out[f"sweep-delaunay-{d}-rep"] = report_dict(sweep(T, workers=WORKERS))
    for d in range(1, 5):
        T = builtin(f"delaunay-{d}")
        out[f"sweep-delaunay-{d}-raw"] = report_dict(
            sweep(T, raw_space=True, workers=WORKERS)
        )
    T3 = builtin("delaunay-3")
    out["sweep-delaunay-3-40-100"] = report_dict(sweep(T3, SweepRange(40, 100)))
    out["sweep-delaunay-3-0-40"] = report_dict(sweep(T3, SweepRange(0, 40)))
    out["sweep-delaunay-3-100-128"] = report_dict(sweep(T3, SweepRange(100, 128)))
    out["sweep-delaunay-3-5-5"] = report_dict(sweep(T3, SweepRange(5, 5)))
    T4 = builtin("delaunay-4")
    out["sample-delaunay-4-5000-42"] = report_dict(sample(T4, 5000, seed=42))
    out["sample-delaunay-4-5000-43"] = report_dict(sample(T4, 5000, seed=43))
    out["sample-delaunay-2-1-0"] = report_dict(sample(builtin("delaunay-2"), 1, seed=0))
    out["sample-delaunay-6-100000-66"] = report_dict(
        sample(builtin("delaunay-6"), 100_000, seed=66, workers=WORKERS)
    )
    out["sample-delaunay-7-200000-11"] = report_dict(
        sample(builtin("delaunay-7"), 200_000, seed=11, workers=WORKERS)
    )
    for name in ("bowtie8", "fig2-middle8", "fig2-right8", "delaunay-8"):
        out[f"sample-{name}-50000-20260810"] = report_dict(
            sample(builtin(name), 50_000, seed=20260810, workers=WORKERS)
        )
    out["sample-delaunay-9-20000-9"] = report_dict(
        sample(builtin("delaunay-9"), 20_000, seed=9, workers=WORKERS)
    )
    rng = random.Random(0xC0FFEE)
    for d in (3, 4, 5):
        T = random_unimodular(d, rng)
        r = sweep(T, workers=WORKERS)
        rd = report_dict(r)
        rd["edges"] = edges_flat(T)
        out[f"sweep-random-{d}-rep"] = rd
    lift = {p: 0 for p in lattice_points(3)}
    lift[(1, 1)] = 7
    Ts = from_lifting(3, lift)
    rd = report_dict(sweep(Ts, raw_space=True))
    rd["edges"] = edges_flat(Ts)
    out["sweep-spike-3-raw"] = rd
    T7 = builtin("delaunay-7")
    rd = report_dict(sweep(T7, SweepRange(0, 1 << 16), raw_space=True, workers=WORKERS))
    out["sweep-delaunay-7-raw-0-65536"] = rd
    dump("reports.json", out)


def part_c2():
    t0 = time.time()
    r = sweep(builtin("delaunay-6"), workers=WORKERS)
    out = report_dict(r)
    out["seconds"] = time.time() - t0
    out["workers"] = WORKERS
    dump("c2_delaunay6_rep.json", out)


def part_c3():
    """Sixteen raw slices of 2^20 inside the lower half [0, 2^35) of delaunay-7."""
    T = builtin("delaunay-7")
    c = Classifier(T)
    rng = random.Random(7)
    n = 1 << 20
    offsets = [rng.randrange(0, (1 << 35) - n) for _ in range(16)]
    slices = []
    t0 = time.time()
    for a in offsets:
        r = sweep(T, SweepRange(a, a + n), raw_space=True, workers=WORKERS, classifier=c)
        slices.append({"start": a, "end": a + n, **report_dict(r)})
    dump(
        "c3_delaunay7_raw_slices.json",
        {"slices": slices, "seconds": time.time() - t0, "workers": WORKERS},
    )


def part_c5():
    """sample_kernel draw slices (kernels.py:447-462), seed 20260810, 42 bits."""
    seed = 20260810
    n = 1 << 20
    k0s = [0, 1 << 39, 10**12 - n]
    out = []
    t0 = time.time()
    for name in ("bowtie8", "fig2-middle8", "fig2-right8", "delaunay-8"):
        T = builtin(name)
        c = Classifier(T)
        nbits = 42

        def runner(plan, scr, agg, bits, lo, hi, _seed=seed, _nb=nbits):
            return kernels.sample_kernel(plan, scr, agg, bits, _seed, lo, hi, _nb)

        for k0 in k0s:
            chunks = [(lo, min(lo + 65536, k0 + n)) for lo in range(k0, k0 + n, 65536)]
            schemes, hist, total = sweep_mod._run_chunks(c, False, chunks, WORKERS, runner)
            r = sweep_mod._finish(T, False, schemes, hist, total, {"mode": "sample-slice"})
            out.append({"name": name, "k0": k0, "k1": k0 + n, "seed": seed, **report_dict(r)})
    dump("c5_sample_slices.json", {"slices": out, "seconds": time.time() - t0})


def part_fig():
    """Edge lists of the three degree-8 figure triangulations (package data)."""
    data = {}
    for name in ("bowtie8", "fig2-middle8", "fig2-right8"):
        T = builtin(name)
        data[name] = {"degree": 8, "edges": edges_flat(T), "fingerprint": T.fingerprint()}
    path = os.path.join(
        os.path.dirname(os.path.dirname(OUT)), "paper_2604_09221_b200", "data", "figure8.json"
    )
    with open(path, "w") as fh:
        json.dump(data, fh, separators=(",", ":"), sort_keys=True)
        fh.write("\n")
    print(f"wrote {path}")


def part_large():
    """Per-pair classifications beyond the 64-bit sign word (d = 10..48):
    the reference's Classifier handles any degree (test_acceptance.py:223-253)."""
    rng = random.Random(0x1A4E)
    out = []
    pool = [(f"delaunay-{d}", builtin(f"delaunay-{d}")) for d in (10, 11, 12, 16, 24, 48)]
    for d in (10, 13):
        pool.append((f"random-{d}", random_unimodular(d, rng)))
    for name, T in pool:
        c = Classifier(T)
        d = T.degree
        rows = []
        count = 12 if d >= 24 else 40
        for _ in range(count):
            s = random_bits(d, rng)
            r = c.classify(s)
            rows.append([s, r.scheme, r.oval_count, r.region_count])
        if name.startswith("delaunay-"):
            s = "".join(str((i * j) % 2) for i, j in lattice_points(d))
            r = c.classify(s)
            rows.append([s, r.scheme, r.oval_count, r.region_count])
        out.append({"name": name, "degree": d, "edges": edges_flat(T),
                    "fingerprint": T.fingerprint(), "rows": rows})
    dump("pairs_large.json", out)


PARTS = {
    "large": part_large,
    "tri": part_tri,
    "pairs": part_pairs,
    "garbage": part_garbage,
    "reports": part_reports,
    "fig": part_fig,
    "c2": part_c2,
    "c3": part_c3,
    "c5": part_c5,
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(PARTS)
    for nm in names:
        t = time.time()
        PARTS[nm]()
        print(f"[{nm}] {time.time() - t:.1f}s", flush=True)
