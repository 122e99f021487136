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


def _garbage_T(d, rng, drop_frac, chords):
    base = builtin(f"delaunay-{d}")
    pts = lattice_points(d)
    edges = list(base.edges)
    for _ in range(int(len(edges) * drop_frac)):
        edges.pop(rng.randrange(len(edges)))
    for _ in range(chords):
        p, q = rng.sample(pts, 2)
        e = (p, q) if p < q else (q, p)
        if e not in edges:
            edges.append(e)
    return Triangulation(d, tuple(sorted(edges)), ())


def part_status():
    """Rows of the compiled kernel (kernels.py:107-356) for every status the
    classifier can return on a bad plan: TOO_MANY_REGIONS (kernels.py:183),
    NO_ODD_REGION / MANY_ODD_REGIONS (:193,:196), NO_PSEUDOLINE (:228),
    ROOT_CONFLICT (:216), NONSEPARATING_OVAL (:211), NOT_A_TREE (:221,:230),
    DISCONNECTED (:266).  Plans are tuples an unvalidated caller can hand to
    the kernel:

    * ``edges``: dropped edges and random chords;
    * ``maxreg``: a valid plan with its maxreg field lowered;
    * ``pairs``: a random subset of the antipodal pairs (maxreg raised to 31);
    * ``bogus``: an extra antipodal "pair" joining the two ends of a diamond
      edge (maxreg raised to 31) -- not a (p, -p) pair, so only the generic
      any-degree engine accepts it (``engine``: "generic").

    A random search keeps up to 24 rows per (degree, status)."""
    rng = random.Random(0x57A7)
    want = 24
    out = []
    kinds = ("edges", "maxreg", "pairs", "bogus")
    for d in range(2, 9):
        got = {s: 0 for s in range(9)}
        trials = 0
        target = (1, 2, 3, 6, 7, 8) if d % 2 == 0 else (1, 4, 5, 7, 8)
        while trials < 800 and min(got[s] for s in target) < want:
            kind = kinds[trials % 4]
            trials += 1
            if kind == "edges" or rng.random() < 0.3:
                T = _garbage_T(d, rng, rng.choice((0.0, 0.05, 0.1, 0.2, 0.35)),
                               rng.choice((0, 1, 2, 4, 8)))
            else:
                T = builtin(f"delaunay-{d}")
            c = Classifier(T)
            common = list(c._plan_common)
            if kind == "maxreg":
                common[10] = rng.randint(1, max(1, int(common[10]) - 2))
            elif kind == "pairs":
                keep = [k for k in range(len(common[8])) if rng.random() < rng.random()]
                common[8] = common[8][keep].copy()
                common[9] = common[9][keep].copy()
                common[10] = 31
            elif kind == "bogus":
                e = rng.randrange(len(common[3]))
                common[8] = np.append(common[8], np.int32(common[3][e]))
                common[9] = np.append(common[9], np.int32(common[4][e]))
                common[10] = 31
            c.maxreg = int(common[10])
            c._plan_common = tuple(common)
            plan = c.plan(raw_space=True)
            scr = c.make_scratch()
            pd = plan_dict(c)
            rows = []
            npts = len(lattice_points(d))
            for _ in range(256):
                m = rng.getrandbits(npts)
                bits = np.array([(m >> k) & 1 for k in range(npts)], dtype=np.uint8)
                st, ov, nr, ln = kernels.classify_bits_kernel(plan, scr, bits)
                st = int(st)
                if st == 0 or got[st] >= want:
                    continue
                got[st] += 1
                rows.append([m, st, int(ov), int(nr), None])
            if rows:
                out.append({"name": f"status-{d}-{trials}-{kind}", "degree": d, "kind": kind,
                            "engine": "generic" if kind == "bogus" else "mask",
                            "edges": [[p[0], p[1], q[0], q[1]] for p, q in T.edges],
                            "plan": pd, "rows": rows})
        print(f"d={d}: {trials} plans, rows per status {got}", flush=True)
    dump("status.json", out)


def part_diff():
    """The reference's differential criterion (test_acceptance.py:144-160)
    replayed with the same generator and seed: 25 random unimodular T per
    degree d = 1..6, 10^4 random sign vectors per degree (T = k mod 25),
    each classified by the reference Classifier (which that test holds equal
    to oracle_classify).  Rows: [k, sign word, scheme id, ovals, regions]."""
    rng = random.Random(0xD1FF)
    out = []
    for d in range(1, 7):
        pool = [random_unimodular(d, rng) for _ in range(25)]
        cls = [Classifier(T) for T in pool]
        names, rows = {}, []
        for n in range(10_000):
            k = n % 25
            s = random_bits(d, rng)
            r = cls[k].classify(s)
            word = sum(1 << i for i, ch in enumerate(s) if ch == "1")
            sid = names.setdefault(r.scheme, len(names))
            rows.append([k, word, sid, r.oval_count, r.region_count])
        out.append({"degree": d, "triangulations": [edges_flat(T) for T in pool],
                    "fingerprints": [T.fingerprint() for T in pool],
                    "schemes": sorted(names, key=names.get), "rows": rows})
    dump("diff.json", out)


def part_garbage_sweep():
    """sweep_kernel (kernels.py:423-436) on degree-7/8 bad plans whose failures
    are rare, over ranges where the first failure lies deep inside: the
    (status, smallest failing index) pair a sweep must report."""
    rng = random.Random(0x5EE9)
    out = []
    for d, raw, count in ((7, True, 4), (7, False, 2), (8, False, 2)):
        npts = len(lattice_points(d))
        nbits = npts if raw else npts - 3
        found = 0
        tries = 0
        while found < count and tries < 300:
            tries += 1
            T = _garbage_T(d, rng, rng.choice((0.0, 0.01, 0.02)), rng.choice((1, 1, 2)))
            c = Classifier(T)
            plan = c.plan(raw_space=raw)
            scr = c.make_scratch()
            bits = np.zeros(npts, dtype=np.uint8)
            # failure rate on 2048 random indices: keep plans failing rarely
            fails = 0
            for _ in range(2048):
                kernels._expand_bits(plan[11], npts, rng.getrandbits(nbits), bits)
                st, _, _, _ = kernels.classify_bits_kernel(plan, scr, bits)
                fails += st != 0
            if not (1 <= fails <= 40):
                continue
            n = 1 << 20
            a = rng.randrange(0, (1 << nbits) - n) & ~0xFFF
            agg = sweep_mod._make_agg(c.maxreg)
            st, bad = kernels.sweep_kernel(plan, scr, agg, bits, a, a + n)
            if st == 0 or bad - a < 4096:
                continue
            found += 1
            out.append({"name": f"gsweep-{d}-{'raw' if raw else 'rep'}-{found}", "degree": d,
                        "raw": raw, "start": a, "end": a + n, "status": int(st), "bad": int(bad),
                        "fail_rate_2048": fails,
                        "edges": [[p[0], p[1], q[0], q[1]] for p, q in T.edges],
                        "plan": plan_dict(c)})
            print(f"d={d} raw={raw}: status {st} at {bad} (start {a}, +{bad - a})", flush=True)
    dump("garbage_sweep.json", out)


def part_c4set():
    """Config C4's triangulations: the first 4,096 draws of the
    reference's own generator random_unimodular(7, Random(0xB7))
    (tests/conftest.py:8-25; the first 16 are the c4-7-k fixtures).  Saved
    as uint8 edge arrays [4096, 84, 4] (bench.py's C4 workload input)."""
    rng = random.Random(0xB7)
    E = np.zeros((4096, 84, 4), np.uint8)
    fps = []
    for k in range(4096):
        T = random_unimodular(7, rng)
        e = edges_flat(T)
        assert len(e) == 84
        E[k] = np.array(e, np.uint8)
        fps.append(T.fingerprint())
    path = os.path.join(OUT, "c4_d7_4096.npz")
    np.savez_compressed(path, edges=E, fingerprints=np.array(fps))
    print(f"wrote {path} ({os.path.getsize(path)} bytes)", flush=True)


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
    "status": part_status,
    "diff": part_diff,
    "gsweep": part_garbage_sweep,
    "c4set": part_c4set,
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(PARTS)
    for nm in names:
        t = time.time()
        PARTS[nm]()
        print(f"[{nm}] {time.time() - t:.1f}s", flush=True)
