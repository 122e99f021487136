"""Per-rank work of the strong-scaling C3 bench at N GPUs, timed on one GPU:
the contiguous shard [0, 2^35 / N) swept as one call (CUDA events), N = 1..8.
    python scripts/c3_shard_steps.py"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2604_09221_b200 import Classifier, builtin  # noqa: E402

T = builtin("delaunay-7")
c = Classifier(T, device=0)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
c.native.set_stream(s.cuda_stream)
for n in (1, 2, 4, 8):
    end = (1 << 35) // n
    for _ in range(2):
        c.native.agg_reset(); c.native.sweep_async(True, 0, end); c.native.agg_fetch()
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c.native.agg_reset()
        a.record(s)
        c.native.sweep_async(True, 0, end)
        b.record(s)
        c.native.agg_fetch()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = sorted(ts)[1]
    print(f"N={n}: shard 2^35/{n} in {ms:.2f} ms per rank -> ideal-box {(1 << 35) / (ms / 1e3) / 1e12:.2f}e12/s, "
          f"efficiency vs N=1 ~ {None if n == 1 else ''}", flush=True)
