#!/usr/bin/env python3
"""Headline benchmark: patchworks classified per second, degree-7 full sign
enumeration (BASELINE.json metric, config C3), 1..N B200.

Workload (config C3): T = delaunay-7 (the staircase), raw index space,
lower half [0, 2^35) = the 2^36 sign space modulo the global sign flip
(SURVEY.md section 0.1).  A step is one slice of 2^34 consecutive indices
per GPU (weak scaling: rank r of N sweeps slice s*N + r); at N=1 the
default 2 timed steps are the complete enumeration.  Indices are generated
on the device (there is no input tensor), so `value` is kernel-resident
throughput; `e2e` runs the same slices through the public API
(`paper_2604_09221_b200.sweep`), host round trip and string rendering
included.

`--impl reference` times the reference algorithm on the host cores instead
(the plain-C restatement in oracle/, all threads), same metric and config,
each step a bounded 2^21-index slice.
"""

from __future__ import annotations

import argparse
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
W_D = {4: 249, 5: 381, 6: 541, 7: 729, 8: 945, 9: 1189}  # 2|E_diamond| + |V_diamond|
CLOCK_FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def ncu_traffic(kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel`, from the
    committed ncu --set full capture (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f)[kernel]["dram_bytes_per_launch"]
    except (OSError, KeyError, ValueError):
        return None


def ncu_kernel(kernel):
    """Issue / pipe utilisation of `kernel` from the committed ncu capture, or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)[kernel]
        return {k: v for k, v in d.items() if k != "dram_bytes_per_launch"}
    except (OSError, KeyError, ValueError):
        return None


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            p = json.load(fh)
        return float(p.get("sm_max_mhz", 1965.0)), "MEASURED_PEAKS.json sm_max_mhz"
    except (OSError, ValueError):
        return 1965.0, "fallback 1965 MHz (B200_PROFILING.md clocks.max.sm)"


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


def oracle_rate(n_per_slice: int, slices: int, threads: int, seed: int = 7):
    """The reference algorithm (plain-C restatement, oracle/) on host cores."""
    from oracle import oracle as O
    from paper_2604_09221_b200 import builtin
    from paper_2604_09221_b200.diamond import plan_arrays, reflect

    plan = O.OraclePlan.from_arrays(plan_arrays(reflect(builtin(f"delaunay-{DEGREE}"))))
    rng = random.Random(seed)
    O.sweep(plan, True, 0, 1 << 14, threads=threads)  # warm
    total, elapsed = 0, 0.0
    for _ in range(slices):
        a = rng.randrange(0, DOMAIN - n_per_slice)
        t0 = time.perf_counter()
        r = O.sweep(plan, True, a, a + n_per_slice, threads=threads)
        elapsed += time.perf_counter() - t0
        assert r["status"] == 0 and r["total"] == n_per_slice
        total += n_per_slice
    return total / elapsed, total, elapsed


def run_reference(args, rank, world):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    n = 1 << 21
    rng = random.Random(11)
    from oracle import oracle as O
    from paper_2604_09221_b200 import builtin
    from paper_2604_09221_b200.diamond import plan_arrays, reflect

    plan = O.OraclePlan.from_arrays(plan_arrays(reflect(builtin(f"delaunay-{DEGREE}"))))
    offs = [rng.randrange(0, DOMAIN - n) for _ in range(args.warmup + args.steps)]
    for a in offs[:args.warmup]:
        O.sweep(plan, True, a, a + n, threads=threads)
    t0 = time.perf_counter()
    for a in offs[args.warmup:]:
        r = O.sweep(plan, True, a, a + n, threads=threads)
        assert r["status"] == 0
    dt = time.perf_counter() - t0
    value = n * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "patchworks/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic (sign indices)",
        "config": {"workload": "C3 delaunay-7 raw lower half [0,2^35); bounded 2^21-index "
                               "slices at random offsets", "degree": DEGREE,
                   "parallelism": f"{threads} host threads"},
        "cpu_baseline": {"value": value, "unit": "patchworks/s", "cores": threads,
                         "kind": "port", "cpu": cpu_model(),
                         "sample": f"{args.steps} x 2^21 raw indices at random offsets "
                                   "(Random(11)); oracle/tcg_oracle.c restates kernels.py"},
        "e2e": {"value": value, "unit": "patchworks/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2604_09221_b200 import Classifier, SweepRange, builtin, merge, sweep
    from paper_2604_09221_b200.distributed import allreduce_aggregate
    from paper_2604_09221_b200.sweep import report_from_agg

    # one process per GPU; BENCH_BACKEND=gloo lets a 2-rank run share one GPU
    # (used to exercise the N>1 path on a single-GPU box; ranks never wait
    # on each other inside a kernel)
    gpu = local_rank % torch.cuda.device_count()
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    coll_dev = dev if BACKEND == "nccl" else torch.device("cpu")
    T = builtin(f"delaunay-{DEGREE}")
    c = Classifier(T, device=gpu)
    # a dedicated stream: the library and the timing events must share it
    # (handle 0 would mean "the plan's own stream" to tcg_plan_set_stream)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    c.native.set_stream(stream.cuda_stream)
    sl = 1 << args.slice_log2

    def rng_of(step):
        a = (args.offset + (step * world + rank) * sl) % DOMAIN
        a -= a % sl
        return a, a + sl

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    # ---- warm-up (untimed): same launches as a timed step, L2 flush included
    for s in range(args.warmup):
        flush.zero_()
        a, b = rng_of(args.steps + s)
        c.native.agg_reset()
        c.native.sweep_async(True, a, b)
        c.native.agg_fetch()
    torch.cuda.synchronize()

    # ---- timed: K steps, device events, max over ranks
    gpu_index = gpu
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        try:
            gpu_index = int(vis.split(",")[local_rank])
        except (ValueError, IndexError):
            pass
    hist_acc = np.zeros(64, np.int64)
    tables = []
    k_ms = []
    launches0 = c.native.launches()
    c.native.kernel_times()  # clear
    c.native.tile_stats()  # clear
    c.native.level2_stats()  # clear
    c.native.set_timing(True)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(gpu_index) as clocks:
        barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        step_ev = []
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
            h, tot, keys, counts, wits = agg.result()
            hist_acc += np.asarray(h, np.int64)
            tables.append((keys, counts, wits))
            k_ms.append((ka, kb))
            sb = torch.cuda.Event(enable_timing=True)
            sb.record(stream)
            step_ev.append((sa, sb))
        from paper_2604_09221_b200.distributed import merge_tables

        keys, counts, wits = merge_tables(tables)
        hist, total, keys, counts, wits = allreduce_aggregate(
            hist_acc.tolist(), int(hist_acc.sum()), keys, counts, wits,
            device=coll_dev if world > 1 else None)
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
    # dominant kernel: the kind with the most device time
    dom = max(ktimes, key=lambda k: ktimes[k][0])
    dom_ms, dom_n = ktimes[dom]
    log("kernel ms by kind:", {k: round(v[0], 2) for k, v in ktimes.items() if v[1]})
    t = torch.tensor([ms, dom_ms, statistics.mean(kern)], dtype=torch.float64, device=coll_dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max, dom_ms_max, sweep_ms = float(t[0]), float(t[1]), float(t[2])
    units = args.steps * sl * world
    value = units / (ms_max / 1e3)
    report = report_from_agg(T, True, hist, total, keys, counts, wits, {})
    assert report.total_classified == units

    # ---- e2e through the public API (host round trip + string rendering)
    def e2e_step(s):
        a, b = rng_of(s)
        return sweep(T, SweepRange(a, b), raw_space=True, classifier=c)

    e2e_step(args.steps)  # warm the path
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = None
    for s in range(args.steps):
        r = e2e_step(s)
        rep = r if rep is None else merge(rep, r)
    if world > 1:
        from paper_2604_09221_b200.io import report_jsonl  # noqa: F401
        gathered = [None] * world
        dist.all_gather_object(gathered, (rep.oval_histogram, rep.scheme_map,
                                          rep.total_classified))
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    te = torch.tensor([e2e_s], dtype=torch.float64, device=coll_dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = units / float(te[0])
    consistent = (world > 1) or (rep.scheme_map == report.scheme_map and
                                 rep.oval_histogram == report.oval_histogram)

    if rank != 0:
        return
    # ---- parity spot check against reference slices (tests/golden, committed)
    parity = None
    gpath = os.path.join(ROOT, "tests", "golden", "c3_delaunay7_raw_slices.json")
    if os.path.exists(gpath):
        with open(gpath) as fh:
            gs = json.load(fh)["slices"]
        ok = 0
        for g in gs:
            r = sweep(T, SweepRange(g["start"], g["end"]), raw_space=True, classifier=c)
            ok += (list(r.oval_histogram) == g["hist"] and
                   r.scheme_map == {k: tuple(v) for k, v in g["schemes"].items()})
        parity = f"{ok}/{len(gs)} reference C3 slices (2^20 each) bit-exact"

    mhz, peak_src = peaks()
    nsm = c.native.info["sms"]
    peak = nsm * 128 * mhz * 1e6  # thread-instruction issue slots / s / GPU
    # patchworks the classify kernels classified explicitly (the rest are
    # counted through the multiplicities of identical tiles / level-2 records)
    if l2_built:  # level 2 ran: 32 patchworks per level-2 record + level-1 leftovers
        classified_pw = (l2_classified << 5) + (l1_left << tile_bits)
    else:
        classified_pw = tiles_classified << tile_bits if tiles_classified else args.steps * sl
    # achieved = patchworks/s x W(d) per GPU over the issue peak
    achieved = value / world * W_D[DEGREE]
    kernel_names = {"tile_classify": "k_tile_classify<K=4,odd,raw>",
                    "enumerate": "k_enumerate<K=4,odd,raw>",
                    "tile_build": "k_tile_from_super", "tile_dedup": "k_tile_dedup",
                    "l2_build": "k_l2_from_l15 (+ k_l2_build)", "l2_dedup": "k_l2_dedup",
                    "l2_classify": "k_l2_classify", "batch": "k_batch",
                    "super_build": "k_super_build<K=4,raw>", "l15_build": "k_l15_build",
                    "l15_dedup": "k_l2_dedup (stage 1)"}
    total_kernel_ms = sum(v[0] for v in ktimes.values())
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        rate, n_cpu, sec = oracle_rate(1 << 22, 4, threads)
        cpu = {"value": rate, "unit": "patchworks/s", "cores": threads, "kind": "port",
               "cpu": cpu_model(),
               "sample": f"4 x 2^22 delaunay-7 raw indices at random offsets (Random(7)), "
                         f"{n_cpu} patchworks in {sec:.1f} s; oracle/tcg_oracle.c restates "
                         "the reference kernels.py on all host threads"}
    d2h = 4 + 4 + 512 + 8 + 24 * len(report.scheme_map)
    line = {
        "metric": METRIC, "value": value, "unit": "patchworks/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic: exhaustive sign-index enumeration, indices generated on device",
        "config": {
            "workload": "C3: delaunay-7 raw sweep, lower half [0,2^35) = 2^36 mod global "
                        f"sign flip; 2^{args.slice_log2} indices per GPU per step",
            "degree": DEGREE, "triangulation": "delaunay-7 (staircase)", "domain": "raw",
            "parallelism": f"dp{world}", "l2": "flushed between steps (256 MiB write)",
            "covered": f"{units} indices = {units / DOMAIN:.3f} of the 2^35 domain",
        },
        "roofline": {
            "bound": "issue", "achieved": achieved, "peak": peak, "unit": "elem-visits/s",
            "frac": achieved / peak, "traffic": ncu_traffic(kernel_names[dom]),
            "note": f"SURVEY 8(d) integer-issue roofline (no tensor or HBM-bound work): "
                    f"achieved = patchworks/s per GPU x W(7) = 2|E|+|V| = 729 element visits "
                    f"(the reference algorithm's work per patchwork); peak = {nsm} SMs x 128 "
                    f"lanes x {mhz:.0f} MHz ({peak_src}). frac > 1 means the path does less "
                    f"than W(7) work per patchwork: super-tile/tile contraction plus exact "
                    f"deduplication classify 1 patchwork in "
                    f"{(args.steps * sl / classified_pw) if classified_pw else 0:.0f} explicitly. "
                    f"kernel = the kind with the most CUDA-event time ({dom}); its hardware "
                    "issue utilisation and dram bytes per launch come from the committed ncu "
                    "capture (profiles/ncu_traffic.json)",
            "kernel": kernel_names[dom], "kernel_ms": dom_ms_max / max(1, dom_n),
            "launches": dom_n,
            "share_of_device_time": dom_ms / total_kernel_ms if total_kernel_ms else None,
            "kernel_ncu": ncu_kernel(kernel_names[dom]),
            "kernels_ms": {k: round(v[0], 3) for k, v in ktimes.items()},
            "sweep_ms_per_step": sweep_ms,
            "dedup": {"tiles": tiles_built, "distinct_tiles": tiles_classified,
                      "level2_records": l2_built, "level2_distinct": l2_classified,
                      "level1_leftover_tiles": l1_left,
                      "patchworks_classified": classified_pw,
                      "factor": args.steps * sl / classified_pw if classified_pw else None,
                      "note": "identical contracted tiles, then identical level-2 records "
                              "(32 patchworks each), are classified once and counted with "
                              "their multiplicity (exact; within each chunk of up to 2^34 "
                              "indices of one sweep call; never across steps)"},
        },
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "patchworks/s", "h2d_bytes_per_step": 16,
                "d2h_bytes_per_step": d2h,
                "path": "paper_2604_09221_b200.sweep(T, SweepRange(a,b), raw_space=True) per "
                        "step + merge; h2d = the (start,end) pair, d2h = aggregate"},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "distinct_schemes": len(report.scheme_map),
        "max_ovals": report.max_ovals(),
        "consistent_e2e_vs_device": consistent,
        "parity": parity,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--slice-log2", type=int, default=34)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--offset", type=lambda x: int(x, 0), default=0,
                    help="first index of the timed slices (profiling away from the easy low prefix)")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warning: the contract asks for >= 3 warm-up steps")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
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
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
