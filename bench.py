#!/usr/bin/env python3
"""Headline benchmark: patchworks classified per second, degree-7 full sign
enumeration (BASELINE.json metric, config C3), on 1..N B200.

Workload (config C3, BASELINE.json configs[2]): T = delaunay-7 (the
staircase), raw index space, lower half [0, 2^35) = the 2^36 sign space
modulo the global sign flip.  One step = the COMPLETE enumeration: the
2^35 indices are split into N contiguous shards, one per GPU (strong
scaling: the total work is fixed); a rank sweeps its shard as one call
(the library's deduplication window is up to 2^35 indices, so at N = 1 the
whole domain is one window), then the per-rank aggregates are merged (NCCL
all_reduce + all_gather, a few KB).  Every step's merged report is checked
against the full C3 report computed by the pinned CPU oracle
(tests/golden/c3_full.json) and the reference's own 2^20-index slices; a
mismatch makes the run exit 1.

`value` is device-resident throughput (indices are generated on the
device); `e2e` runs the same steps through the public API (`sweep`, or
`distributed.sweep_sharded` for N > 1) with the host round trip.
`--weak` keeps the per-GPU work fixed instead (2^33 indices per GPU per
step at disjoint offsets of the raw 2^36 space).

`--impl reference` times the reference's own CPU implementation (`tcurves`,
installed from /root/reference into baseline/_ref) on all host cores, same
metric and config, each step a bounded 2^22-index slice at a random offset.

By default (N = 1) the line also carries `other_workloads`: config C5
(random sampling, degree 8: bowtie8, delaunay-8, fig2-middle8, fig2-right8,
through the separator-split sampler, with the reference's own sampler on the
host cores as cpu_baseline) and config C4 (4,096 random degree-7
triangulations x 2^16 signs, the per-patchwork full-diamond kernel).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import random
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "patchworks classified/sec, degree-7 full sign enumeration, 1/2/4/8 B200"
BACKEND = os.environ.get("BENCH_BACKEND", "nccl")
DEGREE = 7
DOMAIN = 1 << 35  # raw lower half: one index per global-flip orbit
RAW_DOMAIN = 1 << 36
W_D = {4: 249, 5: 381, 6: 541, 7: 729, 8: 945, 9: 1189}  # 2|E_diamond| + |V_diamond|
CLOCK_FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
# kernel kinds timed by the library (tcg.h TCG_KT_*) -> kernel names in ncu
KIND_KERNELS = {
    "super_build": ["k_super_build", "k_super_dedup"],
    "tile_build": ["k_tile_from_super", "k_tile_build_lanes"],
    "tile_dedup": ["k_tile_dedup", "k_super_prop"], "l15_build": ["k_l15_build"],
    "l15_dedup": ["k_l2_dedup/stage1"], "l2_build": ["k_l2_from_l15", "k_l2_build"],
    "l2_dedup": ["k_l2_dedup/level2"], "l2_classify": ["k_l2_classify", "k_l2_classify_even"],
    "tile_classify": ["k_tile_classify"], "enumerate": ["k_enumerate"], "batch": ["k_batch"],
    "split_build": ["k_split_build"], "sample_split": ["k_sample_split"],
    "sample_list": ["k_sample_list"],
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def source_sha16():
    """sha256 of the CUDA sources (csrc/*.cu, *.cuh in name order), 16 hex digits."""
    d = os.path.join(ROOT, "paper_2604_09221_b200", "csrc")
    h = hashlib.sha256()
    for f in sorted(os.listdir(d)):
        if f.endswith((".cu", ".cuh")):
            with open(os.path.join(d, f), "rb") as fh:
                h.update(fh.read())
    return h.hexdigest()[:16]


def ncu_profile(name="ncu_kernels.json"):
    """Per-kernel counters of one bench step (N = 1; ncu_kernels.json: C3,
    ncu_kernels_c5.json: 2^26 bowtie8 draws) from the committed ncu capture,
    if it was taken from this very source (profiles/<name>)."""
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            prof = json.load(f)
    except (OSError, ValueError):
        return None, f"profiles/{name} missing"
    if prof.get("tcg_cu_sha16") != source_sha16():
        return None, (f"profiles/{name} is from CUDA sources {prof.get('tcg_cu_sha16')}, "
                      f"this build is {source_sha16()}: not used")
    return prof, f"profiles/{name} (same CUDA sources)"


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    mhz, hbm, src = 1965.0, 6548.0, "fallback (B200_PROFILING.md: 1965 MHz, ~6.5 TB/s copy)"
    try:
        with open(path) as fh:
            p = json.load(fh)
        mhz = float(p.get("sm_max_mhz", mhz))
        for k in ("hbm_gbs", "hbm_copy_gbps", "hbm_gbps"):
            if k in p:
                hbm = float(p[k])
                break
        src = "MEASURED_PEAKS.json"
    except (OSError, ValueError):
        pass
    return mhz, hbm, src


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 50 ms while timing."""

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        if os.environ.get("BENCH_NO_CLOCKS"):
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={CLOCK_FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50", "-i", str(self.gpu)],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = []
        try:
            with open(self.path) as fh:
                for line in fh:
                    f = [x.strip() for x in line.split(",")]
                    if len(f) >= 9 and f[1].replace(".", "").isdigit():
                        rows.append(f)
        except OSError:
            pass
        finally:
            if self.path and os.path.exists(self.path):
                os.remove(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in rows]
        mx = max(float(r[2]) for r in rows)
        load = [s for s in sm if s > 0.5 * mx] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows), "power_w_max": max(float(r[3]) for r in rows
                                                         if r[3].replace(".", "").isdigit())}


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ------------------------------------------------------------------ CPU legs
def import_tcurves():
    """The reference package itself (installed from /root/reference into
    baseline/_ref, git-ignored, travels to the GPU box), or None."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "tcurves")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "tcg_numba"))
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        import tcurves
        return tcurves
    except Exception as exc:  # numba missing on the host, ...
        log(f"tcurves not importable: {exc!r}")
        return None


def tcurves_rate(tc, n, slices, workers, seed):
    """Reference sweep(T, SweepRange(a, a+n), workers, raw_space=True) at
    random offsets of the C3 domain (BASELINE.md §3 / SURVEY §8(d))."""
    T = tc.builtin(f"delaunay-{DEGREE}")
    c = tc.Classifier(T)
    tc.sweep(T, tc.SweepRange(0, 1 << 12), raw_space=True, classifier=c)  # JIT warm-up
    rng = random.Random(seed)
    elapsed = 0.0
    for _ in range(slices):
        a = rng.randrange(0, DOMAIN - n)
        t0 = time.perf_counter()
        r = tc.sweep(T, tc.SweepRange(a, a + n), workers=workers, raw_space=True, classifier=c)
        elapsed += time.perf_counter() - t0
        assert r.total_classified == n
    return n * slices / elapsed, elapsed


def oracle_rate(n, slices, threads, seed=7):
    """The plain-C restatement of the reference kernels (oracle/) on host cores."""
    from oracle import oracle as O
    from paper_2604_09221_b200 import builtin
    from paper_2604_09221_b200.diamond import plan_arrays, reflect

    plan = O.OraclePlan.from_arrays(plan_arrays(reflect(builtin(f"delaunay-{DEGREE}"))))
    rng = random.Random(seed)
    O.sweep(plan, True, 0, 1 << 14, threads=threads)
    elapsed = 0.0
    for _ in range(slices):
        a = rng.randrange(0, DOMAIN - n)
        t0 = time.perf_counter()
        r = O.sweep(plan, True, a, a + n, threads=threads)
        elapsed += time.perf_counter() - t0
        assert r["status"] == 0 and r["total"] == n
    return n * slices / elapsed, elapsed


def cpu_baseline_block():
    threads = os.cpu_count() or 1
    tc = import_tcurves()
    if tc is not None:
        rate, sec = tcurves_rate(tc, 1 << 22, 4, threads, seed=7)
        one, _ = tcurves_rate(tc, 1 << 17, 1, 1, seed=8)
        port, _ = oracle_rate(1 << 22, 4, threads)
        return {"value": rate, "unit": "patchworks/s", "cores": threads, "kind": "reference",
                "cpu": cpu_model(), "one_worker": one, "port_all_cores": port,
                "sample": f"reference tcurves.sweep(delaunay-7, SweepRange(a, a+2^22), "
                          f"workers={threads}, raw_space=True) at 4 random offsets of [0,2^35) "
                          f"(Random(7)), {sec:.1f} s; one_worker = workers=1 on 2^17 indices; "
                          "port_all_cores = oracle/tcg_oracle.c (C restatement) on the same "
                          "slices"}
    rate, sec = oracle_rate(1 << 22, 4, threads)
    return {"value": rate, "unit": "patchworks/s", "cores": threads, "kind": "port",
            "cpu": cpu_model(),
            "sample": f"4 x 2^22 delaunay-7 raw indices at random offsets (Random(7)) in "
                      f"{sec:.1f} s; oracle/tcg_oracle.c restates the reference kernels.py"}


def run_reference(args, rank, world):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    n = 1 << 22
    rng = random.Random(11)
    offs = [rng.randrange(0, DOMAIN - n) for _ in range(args.warmup + args.steps)]
    tc = import_tcurves()
    if tc is not None:
        T = tc.builtin(f"delaunay-{DEGREE}")
        c = tc.Classifier(T)
        tc.sweep(T, tc.SweepRange(0, 1 << 12), raw_space=True, classifier=c)  # JIT

        def step(a):
            r = tc.sweep(T, tc.SweepRange(a, a + n), workers=threads, raw_space=True,
                         classifier=c)
            assert r.total_classified == n
        kind = "reference"
        what = (f"reference tcurves.sweep(delaunay-7, SweepRange(a, a+2^22), workers={threads}, "
                "raw_space=True), one random offset of [0,2^35) per step (Random(11)); "
                "package installed from /root/reference into baseline/_ref")
    else:
        from oracle import oracle as O
        from paper_2604_09221_b200 import builtin
        from paper_2604_09221_b200.diamond import plan_arrays, reflect

        plan = O.OraclePlan.from_arrays(plan_arrays(reflect(builtin(f"delaunay-{DEGREE}"))))

        def step(a):
            r = O.sweep(plan, True, a, a + n, threads=threads)
            assert r["status"] == 0
        kind = "port"
        what = ("baseline/_ref missing: oracle/tcg_oracle.c (C restatement of kernels.py) on "
                f"{threads} threads, 2^22 indices per step at random offsets (Random(11))")
    for a in offs[:args.warmup]:
        step(a)
    t0 = time.perf_counter()
    for a in offs[args.warmup:]:
        step(a)
    dt = time.perf_counter() - t0
    value = n * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "patchworks/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic (sign indices)",
        "config": {"workload": "C3 delaunay-7 raw lower half [0,2^35); bounded 2^22-index "
                               "slices at random offsets", "degree": DEGREE,
                   "parallelism": f"{threads} host threads"},
        "cpu_baseline": {"value": value, "unit": "patchworks/s", "cores": threads, "kind": kind,
                         "cpu": cpu_model(), "sample": what},
        "e2e": {"value": value, "unit": "patchworks/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- parity checks
def c3_golden():
    """Full C3 report (hist, scheme -> (count, witness)) from the oracle pieces."""
    path = os.path.join(ROOT, "tests", "golden", "c3_full.json")
    try:
        with open(path) as fh:
            doc = json.load(fh)
    except (OSError, ValueError):
        return None
    pieces = doc["pieces"]
    if len(pieces) != DOMAIN >> doc["piece_log2"]:
        return None
    hist = None
    schemes = {}
    for p in pieces.values():
        hist = p["hist"] if hist is None else [a + b for a, b in zip(hist, p["hist"])]
        for s, (c, w) in p["schemes"].items():
            schemes[s] = (schemes[s][0] + c, min(schemes[s][1], w)) if s in schemes else (c, w)
    return hist, schemes


def slice_parity(T, c):
    from paper_2604_09221_b200 import SweepRange, sweep

    with open(os.path.join(ROOT, "tests", "golden", "c3_delaunay7_raw_slices.json")) as fh:
        gs = json.load(fh)["slices"]
    ok = 0
    for g in gs:
        r = sweep(T, SweepRange(g["start"], g["end"]), raw_space=True, classifier=c)
        ok += (list(r.oval_histogram) == g["hist"] and
               r.scheme_map == {k: tuple(v) for k, v in g["schemes"].items()})
    return ok, len(gs)


# ------------------------------------------------------------ other configs
def bench_c5(dev, steps, warmup):
    """Config C5: uniform sampling over the degree-8 representative space
    (seed 20260810, draws k0 = 2^39 ..): the separator-split sampler
    (k_sample_split, csrc/split.cuh; draws it leaves go to k_sample_list)."""
    import torch

    from paper_2604_09221_b200 import Classifier, builtin
    from paper_2604_09221_b200.sweep import report_from_agg, sample_slice

    with open(os.path.join(ROOT, "tests", "golden", "c5_sample_slices.json")) as fh:
        gold = json.load(fh)["slices"]
    out = {}
    n = 1 << 28
    k0 = 1 << 39
    seed = 20260810
    tc = import_tcurves()
    threads = os.cpu_count() or 1
    for name in ("bowtie8", "delaunay-8", "fig2-middle8", "fig2-right8"):
        T = builtin(name)
        c = Classifier(T, device=dev.index)
        stream = torch.cuda.Stream(device=dev)  # events and kernels on one stream
        torch.cuda.set_stream(stream)
        c.native.set_stream(stream.cuda_stream)
        c.native.set_timing(True)
        for s in range(warmup):  # the first one builds the split tables
            c.native.agg_reset()
            c.native.sample_async(seed, k0 + (s + 1) * n * 4, k0 + (s + 1) * n * 4 + n, 42)
            c.native.agg_fetch()
        torch.cuda.synchronize()
        build_ms = c.native.kernel_times()["split_build"][0]
        c.native.split_stats()
        evs = []
        c.native.set_timing(True)
        c.native.kernel_times()
        for s in range(steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c.native.agg_reset()
            a.record(stream)
            c.native.sample_async(seed, k0 + s * n, k0 + (s + 1) * n, 42)
            b.record(stream)
            rc, bad, agg = c.native.agg_fetch()
            assert rc == 0, (rc, bad)
            evs.append((a, b))
        torch.cuda.synchronize()
        kt = c.native.kernel_times()
        c.native.set_timing(False)
        sst = c.native.split_stats()  # state, draws, left to the flat kernel, F vertices, bytes
        ms = sum(x.elapsed_time(y) for x, y in evs) / steps
        t0 = time.perf_counter()
        for s in range(steps):
            sample_slice(T, seed, k0 + s * n, k0 + (s + 1) * n, classifier=c)
        e2e = n * steps / (time.perf_counter() - t0)
        ok = 0
        slices = [g for g in gold if g["name"] == name]
        for g in slices:
            r = sample_slice(T, g["seed"], g["k0"], g["k1"], classifier=c)
            ok += (list(r.oval_histogram) == g["hist"] and
                   r.scheme_map == {k: tuple(v) for k, v in g["schemes"].items()})
        split = sst[0] == 1
        # CPU baseline: the reference's own sampler on all host cores
        cpu = None
        if tc is not None:
            tT = tc.builtin(name)
            tcl = tc.Classifier(tT)
            tc.sample(tT, 1 << 12, seed, workers=threads, classifier=tcl)  # JIT
            ncpu = 1 << 20
            t0 = time.perf_counter()
            r = tc.sample(tT, ncpu, seed, workers=threads, classifier=tcl)
            sec = time.perf_counter() - t0
            assert r.total_classified == ncpu
            cpu = {"value": ncpu / sec, "unit": "draws/s", "cores": threads, "kind": "reference",
                   "sample": f"tcurves.sample({name}, 2^20, seed {seed}, workers={threads}), "
                             f"{sec:.1f} s"}
        kern_ms = (kt["sample_split"][0] + kt["sample_list"][0] if split else kt["enumerate"][0]) / steps
        roof = None
        if split and name == "bowtie8":  # the captured configuration
            prof, psrc = ncu_profile("ncu_kernels_c5.json")
            mhz, _, _ = peaks()
            p_issue = c.native.info["sms"] * 128 * mhz * 1e6
            roof = {"bound": "issue", "unit": "thread-inst/s", "peak": p_issue,
                    "kernel": "k_sample_split", "source": psrc, "achieved": None, "frac": None}
            kp = (prof or {}).get("kernels", {}).get("k_sample_split")
            if kp:
                draws = prof.get("draws", 1 << 26)
                per_draw = kp["thread_inst_per_step"] / draws
                split_ms = kt["sample_split"][0] / steps
                roof["achieved"] = per_draw * n / (split_ms / 1e3)
                roof["frac"] = roof["achieved"] / p_issue
                roof["thread_inst_per_draw"] = per_draw
                roof["dram_bytes_per_draw"] = kp["dram_bytes_per_step"] / draws
                roof["ncu"] = {k: v for k, v in kp.items()
                               if k in ("issue_active_pct", "alu_pipe_pct", "threads_per_inst",
                                        "local_sectors_per_step", "registers", "warps_active_pct")}
        out[f"c5_{name}"] = {
            "roofline": roof,
            "metric": "draws classified/sec (degree-8 uniform sampling, one B200)",
            "value": n / (ms / 1e3), "unit": "draws/s", "ms_per_step": ms,
            "e2e": {"value": e2e, "unit": "draws/s", "h2d_bytes_per_step": 32,
                    "path": "sweep.sample_slice (host round trip + string rendering)"},
            "config": {"workload": f"C5 {name}: draws [2^39 + s 2^28, +2^28) seed 20260810, "
                                   "m = splitmix64 & (2^42-1)", "draws_per_step": n},
            "kernel": ("k_sample_split<even> + k_sample_list<6,even>" if split
                       else "k_enumerate<6,even,SAMPLE>"),
            "kernel_ms_per_step": kern_ms,
            "split": {"separator_vertices": sst[3], "table_bytes": sst[4],
                      "table_build_ms": build_ms,
                      "flat_fallback_fraction": sst[2] / sst[1] if sst[1] else None,
                      "sample_split_ms_per_step": kt["sample_split"][0] / steps,
                      "sample_list_ms_per_step": kt["sample_list"][0] / steps} if split else None,
            "parity": f"{ok}/{len(slices)} reference sample_kernel slices (2^20 draws) bit-exact",
            "parity_ok": ok == len(slices),
            "cpu_baseline": cpu,
        }
    return out


def bench_c2(dev, steps, warmup):
    """Config C2: delaunay-6, the exhaustive raw 2^28 sign space per step
    (tile pipeline, even degree); parity: the raw histogram and scheme counts
    are 8x the reference's full representative sweep (tests/golden, the
    (Z/2)^3 symmetry of SURVEY A16), and a representative 2^25 sweep equals it
    bit for bit (witnesses included)."""
    import torch

    from paper_2604_09221_b200 import Classifier, SweepRange, builtin, sweep

    with open(os.path.join(ROOT, "tests", "golden", "c2_delaunay6_rep.json")) as fh:
        g = json.load(fh)
    T = builtin("delaunay-6")
    c = Classifier(T, device=dev.index)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    c.native.set_stream(stream.cuda_stream)
    n = 1 << 28
    for _ in range(warmup):
        c.native.agg_reset()
        c.native.sweep_async(True, 0, n)
        c.native.agg_fetch()
    torch.cuda.synchronize()
    evs = []
    for _ in range(steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c.native.agg_reset()
        a.record(stream)
        c.native.sweep_async(True, 0, n)
        b.record(stream)
        rc, bad, agg = c.native.agg_fetch()
        assert rc == 0, (rc, bad)
        evs.append((a, b))
    torch.cuda.synchronize()
    ms = sum(x.elapsed_time(y) for x, y in evs) / steps
    t0 = time.perf_counter()
    for _ in range(steps):
        r = sweep(T, SweepRange(0, n), raw_space=True, classifier=c)
    e2e = n * steps / (time.perf_counter() - t0)
    raw_ok = (list(r.oval_histogram) == [8 * x for x in g["hist"]] and
              {k: v[0] for k, v in r.scheme_map.items()} ==
              {k: 8 * v[0] for k, v in g["schemes"].items()})
    rep = sweep(T, SweepRange(0, 1 << 25), classifier=c)
    rep_ok = (list(rep.oval_histogram) == g["hist"] and
              rep.scheme_map == {k: tuple(v) for k, v in g["schemes"].items()})
    return {"c2": {
        "metric": "patchworks classified/sec, degree-6 full raw sign enumeration, one B200",
        "value": n / (ms / 1e3), "unit": "patchworks/s", "ms_per_step": ms,
        "e2e": {"value": e2e, "unit": "patchworks/s", "h2d_bytes_per_step": 16,
                "path": "sweep(T, SweepRange(0, 2^28), raw_space=True)"},
        "config": {"workload": "C2: delaunay-6 raw [0, 2^28) (the full 2^28 raw space)",
                   "patchworks_per_step": n},
        "parity": f"raw = 8 x the reference's full representative sweep: {raw_ok}; "
                  f"representative 2^25 sweep bit-exact: {rep_ok}",
        "parity_ok": raw_ok and rep_ok,
    }}


def bench_c4(dev, steps, warmup):
    """Config C4: 4,096 random regular unimodular degree-7 triangulations
    (reference generator, Random(0xB7)) x 2^16 sign words each,
    m = splitmix64(7, k) & (2^36 - 1), one topology per CTA."""
    import numpy as np

    from paper_2604_09221_b200 import MultiClassifier, scheme_from_key
    from paper_2604_09221_b200.lattice import Triangulation

    data = np.load(os.path.join(ROOT, "tests", "golden", "c4_d7_4096.npz"))
    E = data["edges"].astype(int)
    Ts = [Triangulation(7, tuple(((int(a), int(b)), (int(c), int(d))) for a, b, c, d in e), ())
          for e in E]
    mc = MultiClassifier(Ts, device=dev.index)
    per = 1 << 16
    ntri = len(Ts)
    n = ntri * per
    k = np.arange(n, dtype=np.uint64)
    z = np.uint64(7) + (k + np.uint64(1)) * np.uint64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    words = (z ^ (z >> np.uint64(31))) & np.uint64((1 << 36) - 1)
    tri = (np.arange(n, dtype=np.int64) // per).astype(np.int32)
    for _ in range(warmup):
        mc.classify_words(tri, words)
    kms, wall = [], []
    for _ in range(steps):
        t0 = time.perf_counter()
        keys, ov, nr, st = mc.classify_words(tri, words)
        wall.append(time.perf_counter() - t0)
        kms.append(mc.native.last_ms())
    assert (st == 0).all()
    # parity: the 16 c4-7-k fixtures (reference pairs) are the first 16 T
    with open(os.path.join(ROOT, "tests", "golden", "pairs.json")) as fh:
        pairs = {e["name"]: e["rows"] for e in json.load(fh)}
    ok = tot = 0
    ptri, pw, want = [], [], []
    for t in range(16):
        for s, scheme, o, r in pairs[f"c4-7-{t}"]:
            ptri.append(t)
            pw.append(int(s[::-1], 2))
            want.append((scheme, o, r))
    pk, po, pr, ps = mc.classify_words(np.array(ptri, np.int32), np.array(pw, np.uint64))
    for i, (scheme, o, r) in enumerate(want):
        tot += 1
        ok += (ps[i] == 0 and scheme_from_key(int(pk[i]), True) == scheme and
               int(po[i]) == o and int(pr[i]) == r)
    ms = statistics.median(kms)
    return {"c4": {
        "metric": "(triangulation, sign) pairs classified/sec, degree 7, one B200",
        "value": n / (ms / 1e3), "unit": "pairs/s", "ms_per_step": ms,
        "e2e": {"value": n / statistics.median(wall), "unit": "pairs/s",
                "h2d_bytes_per_step": 12 * n, "d2h_bytes_per_step": 14 * n,
                "path": "MultiClassifier.classify_words (host buffers; validation, grouping, pinned-staging pipeline of 2^23-pair chunks)"},
        "config": {"workload": "C4: 4096 T from random_unimodular(7, Random(0xB7)) x 2^16 "
                               "words splitmix64(7,k) & (2^36-1)", "pairs_per_step": n},
        "kernel": "k_multi<4,odd>",
        "parity": f"{ok}/{tot} reference pairs of c4-7-0..15 bit-exact",
        "parity_ok": ok == tot,
    }}


# ---------------------------------------------------------------------- ours
def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2604_09221_b200 import Classifier, SweepRange, builtin, merge, sweep
    from paper_2604_09221_b200.distributed import allreduce_aggregate, shard, sweep_sharded
    from paper_2604_09221_b200.io import report_jsonl
    from paper_2604_09221_b200.sweep import report_from_agg

    # one process per GPU; BENCH_BACKEND=gloo lets a 2-rank run share one GPU
    # (exercises the N>1 path on a single-GPU box; ranks never wait on each
    # other inside a kernel)
    gpu = local_rank % torch.cuda.device_count()
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    coll_dev = dev if BACKEND == "nccl" else torch.device("cpu")
    T = builtin(f"delaunay-{DEGREE}")
    c = Classifier(T, device=gpu)
    # a dedicated stream: the library and the timing events must share it
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    c.native.set_stream(stream.cuda_stream)

    if args.weak:
        sl = 1 << args.slice_log2
        groups = RAW_DOMAIN // (sl * world)
        if groups < 1:
            raise SystemExit(f"--weak: {world} x 2^{args.slice_log2} exceeds the raw 2^36 space")

        def rng_of(step):  # disjoint within a step; the next step takes the next group
            a = ((step % groups) * world + rank) * sl
            return a, a + sl
        units_per_step = sl * world
    else:
        lo, hi = shard(0, DOMAIN, rank, world)

        def rng_of(step):
            return lo, hi
        units_per_step = DOMAIN

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def merged(agg_result):
        h, tot, keys, counts, wits = agg_result
        hist, total, keys, counts, wits = allreduce_aggregate(
            np.asarray(h, np.int64).tolist(), int(tot), keys, counts, wits,
            device=coll_dev if world > 1 else None)
        return report_from_agg(T, True, hist, total, keys, counts, wits, {})

    # ---- warm-up (untimed): same launches as a timed step
    for s in range(args.warmup):
        flush.zero_()
        a, b = rng_of(s + 1)
        c.native.agg_reset()
        c.native.sweep_async(True, a, b)
        c.native.agg_fetch()
    torch.cuda.synchronize()

    gpu_index = gpu
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        try:
            gpu_index = int(vis.split(",")[local_rank])
        except (ValueError, IndexError):
            pass
    launches0 = c.native.launches()
    c.native.kernel_times()  # clear
    c.native.tile_stats()
    c.native.level2_stats()
    c.native.set_timing(True)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    reports, k_ms, step_ev = [], [], []
    with ClockSampler(gpu_index) as clocks:
        barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for s in range(args.steps):
            sa = torch.cuda.Event(enable_timing=True)
            sa.record(stream)
            flush.zero_()  # L2 flush between steps (256 MiB > 126 MB L2)
            a, b = rng_of(s)
            ka = torch.cuda.Event(enable_timing=True)
            kb = torch.cuda.Event(enable_timing=True)
            c.native.agg_reset()
            ka.record(stream)
            c.native.sweep_async(True, a, b)
            kb.record(stream)
            rc, bad, agg = c.native.agg_fetch()
            if rc:
                raise RuntimeError(f"status {rc} at index {bad}")
            reports.append(merged(agg.result()))  # per-step merge over ranks (collective)
            k_ms.append((ka, kb))
            sb = torch.cuda.Event(enable_timing=True)
            sb.record(stream)
            step_ev.append((sa, sb))
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = ev0.elapsed_time(ev1)
    c.native.set_timing(False)
    ktimes = c.native.kernel_times()
    kern = [x.elapsed_time(y) for x, y in k_ms]
    log("step ms:", [round(x.elapsed_time(y), 2) for x, y in step_ev], "kernel ms:",
        [round(k, 2) for k in kern], "total ms:", round(ms, 2))
    launches = c.native.launches() - launches0
    tiles_built, tiles_classified = c.native.tile_stats()
    l2_built, l2_classified, l1_left = c.native.level2_stats()
    tile_bits = c.native.info["tile_bits_raw"]
    dom = max(ktimes, key=lambda k: ktimes[k][0])
    log("kernel ms by kind:", {k: round(v[0], 2) for k, v in ktimes.items() if v[1]})
    t = torch.tensor([ms, statistics.mean(kern)], dtype=torch.float64, device=coll_dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max, sweep_ms = float(t[0]), float(t[1])
    units = args.steps * units_per_step
    value = units / (ms_max / 1e3)
    rank_units = args.steps * (rng_of(0)[1] - rng_of(0)[0])
    for r in reports:
        assert r.total_classified == units_per_step
    deterministic = all(r == reports[0] for r in reports) if not args.weak else True

    # ---- e2e through the public API (host round trip + string rendering)
    def e2e_step(s):
        if args.weak:  # each rank's own slice; reports are per rank
            a, b = rng_of(s)
            return sweep(T, SweepRange(a, b), raw_space=True, classifier=c)
        if world > 1:
            return sweep_sharded(T, 0, DOMAIN, raw_space=True, classifier=c)
        return sweep(T, SweepRange(0, DOMAIN), raw_space=True, classifier=c)

    e2e_step(0)  # warm
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e2e_reports = [e2e_step(s) for s in range(args.steps)]
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    te = torch.tensor([e2e_s], dtype=torch.float64, device=coll_dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = units / float(te[0])
    if args.weak:
        consistent = True
    else:
        consistent = all(r.scheme_map == reports[0].scheme_map and
                         r.oval_histogram == reports[0].oval_histogram for r in e2e_reports)

    # per-rank dedup factor (strong scaling shrinks each rank's window)
    if l2_built:
        classified_pw = (l2_classified << 5) + (l1_left << tile_bits)
    else:
        classified_pw = tiles_classified << tile_bits if tiles_classified else rank_units
    dfac = torch.tensor([rank_units / classified_pw if classified_pw else 0.0],
                        dtype=torch.float64, device=coll_dev)
    dfacs = [torch.zeros_like(dfac) for _ in range(world)]
    if world > 1:
        dist.all_gather(dfacs, dfac)
    else:
        dfacs = [dfac]

    other = {}
    if world == 1 and not args.no_extra:
        other.update(bench_c5(dev, 3, 2))
        other.update(bench_c4(dev, 3, 1))
        other.update(bench_c2(dev, 5, 3))

    if rank != 0:
        return 0
    # ---- parity gate: full report vs the oracle's C3 golden + reference slices
    parity = {}
    ok_all = True
    if not args.weak:
        g = c3_golden()
        if g is not None:
            hist, schemes = g
            full_ok = all(list(r.oval_histogram) == hist[:len(r.oval_histogram)] and
                          r.scheme_map == schemes for r in reports)
            parity["full_c3"] = ("every step's merged report == tests/golden/c3_full.json "
                                 "(pinned oracle, all 2^35 indices)" if full_ok else "MISMATCH")
            ok_all &= full_ok
        else:
            parity["full_c3"] = "tests/golden/c3_full.json incomplete: not checked"
    ok, n_sl = slice_parity(T, c)
    parity["reference_slices"] = f"{ok}/{n_sl} reference C3 slices (2^20 each) bit-exact"
    ok_all &= ok == n_sl and deterministic and consistent
    for k, v in other.items():
        ok_all &= v.get("parity_ok", True)
    rep0 = reports[0]
    rep0.params = {"mode": "sweep", "start": 0, "end": DOMAIN, "raw_space": True}
    parity["report_sha256"] = hashlib.sha256(report_jsonl(rep0).encode()).hexdigest()

    # ---- roofline: dominant kernel's issue rate from a same-source ncu capture
    mhz, hbm_peak, peak_src = peaks()
    nsm = c.native.info["sms"]
    p_issue = nsm * 128 * mhz * 1e6  # thread-instruction issue slots / s / GPU
    prof, prof_src = ncu_profile() if world == 1 and not args.weak else (
        None, "ncu capture is of the N=1 strong step only")
    kms_step = {k: v[0] / args.steps for k, v in ktimes.items() if v[1]}
    total_kernel_ms = sum(kms_step.values())
    roof = {"bound": "issue", "unit": "thread-inst/s", "peak": p_issue,
            "kernel": "/".join(KIND_KERNELS[dom]), "kernel_kind": dom,
            "kernel_ms_per_step": kms_step[dom],
            "launches_per_step": ktimes[dom][1] / args.steps,
            "share_of_device_time": kms_step[dom] / total_kernel_ms if total_kernel_ms else None,
            "kernels_ms_per_step": {k: round(v, 3) for k, v in kms_step.items()},
            "sweep_ms_per_step": sweep_ms, "achieved": None, "frac": None, "traffic": None,
            "source": prof_src}
    if prof is not None:
        kp = prof["kernels"]
        names = KIND_KERNELS[dom]
        inst = sum(kp[n]["thread_inst_per_step"] for n in names if n in kp)
        dram = sum(kp[n]["dram_bytes_per_step"] for n in names if n in kp)
        nl = max(1, ktimes[dom][1] // args.steps)
        roof["achieved"] = inst / (kms_step[dom] / 1e3)
        roof["frac"] = roof["achieved"] / p_issue
        roof["traffic"] = dram / nl
        roof["thread_inst_per_launch"] = inst / nl
        roof["ncu"] = {n: {k: v for k, v in kp[n].items()
                           if k in ("issue_active_pct", "alu_pipe_pct", "threads_per_inst",
                                    "local_sectors_per_step", "registers", "warps_active_pct")}
                       for n in names if n in kp}
        hbm = {}
        step_bytes = 0
        for kind, kms in kms_step.items():
            byts = sum(kp[n]["dram_bytes_per_step"] for n in KIND_KERNELS.get(kind, []) if n in kp)
            step_bytes += byts
            if byts:
                gbps = byts / (kms / 1e3) / 1e9
                hbm[kind] = {"dram_bytes_per_step": byts, "GBps": round(gbps, 1),
                             "frac_of_hbm": round(gbps / hbm_peak, 3)}
        roof["issue_per_kind"] = {
            kind: round(sum(kp[n]["thread_inst_per_step"] for n in KIND_KERNELS.get(kind, [])
                            if n in kp) / (kms / 1e3) / p_issue, 3)
            for kind, kms in kms_step.items() if kms > 0}
        roof["hbm"] = {"peak_GBps": hbm_peak, "per_kind": hbm,
                       "dram_bytes_per_step": step_bytes,
                       "bytes_per_patchwork": step_bytes / units_per_step}
    roof["note"] = (f"integer instruction issue bound (no FP / tensor work; SURVEY 8(d)): "
                    f"achieved = thread instructions the dominant kernel executes per step "
                    f"(ncu smsp__thread_inst_executed.sum, same CUDA sources) / its CUDA-event time "
                    f"per step in this run; peak = {nsm} SMs x 128 lanes x {mhz:.0f} MHz "
                    f"({peak_src}). hbm.per_kind: ncu dram bytes / live time vs the copy peak.")

    work_avoidance = {
        "w_d_ratio": value / world * W_D[DEGREE] / p_issue,
        "dedup_factor_per_rank": [float(x) for x in dfacs],
        "note": "patchworks/s per GPU x W(7) = 2|E|+|V| = 729 element visits / P_issue: the "
                "SURVEY 8(d) algorithmic ratio; > 1 because contraction + exact deduplication "
                "classify one patchwork in dedup_factor explicitly (not a hardware fraction)",
    }
    line = {
        "metric": METRIC, "value": value, "unit": "patchworks/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
        "higher_is_better": True, "scaling": "weak" if args.weak else "strong",
        "vs_baseline": None, "dtype": "u64",
        "data": "synthetic: exhaustive sign-index enumeration, indices generated on device",
        "config": {
            "workload": ("C3: delaunay-7 raw sweep, lower half [0,2^35) = 2^36 mod global sign "
                         "flip; one step = the full enumeration, split in N contiguous shards"
                         if not args.weak else
                         f"C3 weak: 2^{args.slice_log2} raw indices per GPU per step, disjoint "
                         "offsets in the raw 2^36 space"),
            "degree": DEGREE, "triangulation": "delaunay-7 (staircase)", "domain": "raw",
            "parallelism": f"dp{world}", "l2": "flushed between steps (256 MiB write)",
            "indices_per_rank_per_step": rng_of(0)[1] - rng_of(0)[0],
        },
        "roofline": roof,
        "work_avoidance": work_avoidance,
        "dedup": {"tiles": tiles_built, "distinct_tiles": tiles_classified,
                  "level2_records": l2_built, "level2_distinct": l2_classified,
                  "level1_leftover_tiles": l1_left, "patchworks_classified": classified_pw},
        "cpu_baseline": (cpu_baseline_block() if world == 1 and not args.no_cpu_baseline
                         else None),
        "e2e": {"value": e2e_value, "unit": "patchworks/s", "h2d_bytes_per_step": 16,
                "d2h_bytes_per_step": 528 + 24 * len(rep0.scheme_map),
                "path": "paper_2604_09221_b200.sweep(T, SweepRange(0, 2^35), raw_space=True) "
                        "(N > 1: distributed.sweep_sharded); h2d = (start, end), d2h = the "
                        "aggregate"},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "distinct_schemes": len(rep0.scheme_map),
        "max_ovals": rep0.max_ovals(),
        "parity": parity,
        "parity_ok": bool(ok_all),
        "other_workloads": other or None,
    }
    print(json.dumps(line), flush=True)
    return 0 if ok_all else 1


def run_single_workload(args):
    """--workload c2 | c4 | c5: one line for that config (N = 1, for profiling)."""
    import torch

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    res = bench_c5(dev, args.steps, args.warmup) if args.workload == "c5" else bench_c2(
        dev, args.steps, args.warmup) if args.workload == "c2" else bench_c4(
        dev, args.steps, args.warmup)
    for k, v in res.items():
        print(json.dumps({"workload": k, **v}), flush=True)
    return 0 if all(v["parity_ok"] for v in res.values()) else 1


def main():
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["c2", "c3", "c4", "c5"], default="c3")
    ap.add_argument("--weak", action="store_true", help="fixed work per GPU (see docstring)")
    ap.add_argument("--slice-log2", type=int, default=33, help="--weak: indices per GPU-step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the C4 / C5 lines")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warning: the contract asks for >= 3 warm-up steps")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return 0
    if args.workload != "c3":
        return run_single_workload(args)
    if world > 1:
        import torch
        import torch.distributed as dist

        gpu = local_rank % torch.cuda.device_count()
        torch.cuda.set_device(gpu)
        if BACKEND == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", gpu))
        else:
            dist.init_process_group(BACKEND)
    try:
        return run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
