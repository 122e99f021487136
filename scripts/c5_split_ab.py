"""C5 A/B: separator-split sampler vs the flat sampler (same draws, same plan).

    python scripts/c5_split_ab.py [log2 draws] [names...]

Prints per triangulation: draws/s of both paths (CUDA events around the
enqueue on the plan's stream), the split statistics and per-kernel times, and
whether the two aggregates are identical.
"""
import sys
import time

sys.path.insert(0, ".")

import torch  # noqa: E402

from paper_2604_09221_b200 import Classifier, builtin  # noqa: E402


def run(c, split, seed, k0, n):
    c.native.set_split(split)
    c.native.agg_reset()
    c.native.sample_async(seed, k0 - n, k0, 42)  # warm (table build on first use)
    c.native.agg_fetch()
    c.native.split_stats()
    c.native.set_timing(True)
    c.native.kernel_times()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c.native.agg_reset()
    a.record(st)
    c.native.sample_async(seed, k0, k0 + n, 42)
    b.record(st)
    rc, bad, agg = c.native.agg_fetch()
    torch.cuda.synchronize()
    kt = {k: v for k, v in c.native.kernel_times().items() if v[1]}
    c.native.set_timing(False)
    return a.elapsed_time(b), (rc, bad, agg.result()), kt, c.native.split_stats()


def main():
    lg = int(sys.argv[1]) if len(sys.argv) > 1 else 26
    names = sys.argv[2:] or ["bowtie8", "delaunay-8", "fig2-middle8", "fig2-right8"]
    n, seed, k0 = 1 << lg, 20260810, 1 << 39
    for name in names:
        T = builtin(name)
        t0 = time.time()
        c = Classifier(T, device=0)
        stream = torch.cuda.Stream()
        torch.cuda.set_stream(stream)
        c.native.set_stream(stream.cuda_stream)
        ms_s, ra, kta, sta = run(c, True, seed, k0, n)
        ms_f, rb, ktb, _ = run(c, False, seed, k0, n)
        same = ra[0] == rb[0] and ra[1] == rb[1] and all(
            (x == y).all() if hasattr(x, "all") else x == y for x, y in zip(ra[2], rb[2]))
        print(f"{name}: split {n / ms_s / 1e6:.3f}e9 draws/s ({ms_s:.1f} ms)  flat {n / ms_f / 1e6:.3f}e9 "
              f"({ms_f:.1f} ms)  x{ms_f / ms_s:.2f}  identical={same}  stats={sta}  "
              f"kernels={ {k: round(v[0], 2) for k, v in kta.items()} }  setup {time.time() - t0:.1f}s",
              flush=True)


if __name__ == "__main__":
    main()
