"""Per-step, per-kernel-kind device times of the C3 step (the bench's timed
loop without the host report merge): python scripts/c3_steps.py [steps]."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2604_09221_b200 import Classifier, builtin  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 12
timing = len(sys.argv) <= 2 or sys.argv[2] != "0"
T = builtin("delaunay-7")
c = Classifier(T, device=0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
c.native.set_stream(stream.cuda_stream)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for s in range(3):
    c.native.agg_reset()
    c.native.sweep_async(True, 0, 1 << 35)
    c.native.agg_fetch()
c.native.set_timing(timing)
c.native.kernel_times()
for s in range(steps):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c.native.agg_reset()
    a.record(stream)
    c.native.sweep_async(True, 0, 1 << 35)
    b.record(stream)
    c.native.agg_fetch()
    torch.cuda.synchronize()
    kt = c.native.kernel_times()
    print(f"step {s}: {a.elapsed_time(b):7.2f} ms  " +
          " ".join(f"{k}={v[0]:.2f}" for k, v in kt.items() if v[1]), flush=True)
