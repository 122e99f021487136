"""ncu target: exactly one bench step between cudaProfilerStart/Stop.

    ncu --profile-from-start off ... python scripts/profile_step.py [c3|c5]

c3: the full C3 enumeration as bench.py times it at N = 1 (delaunay-7 raw
[0, 2^35), two 2^34-index chunks); c5: 2^26 bowtie8 draws at k0 = 2^39."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_09221_b200 import Classifier, builtin  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "c3"
if what == "c3":
    c = Classifier(builtin("delaunay-7"))
    run = lambda: c.native.sweep_async(True, 0, 1 << 35)  # noqa: E731
else:
    c = Classifier(builtin("bowtie8"))
    run = lambda: c.native.sample_async(20260810, 1 << 39, (1 << 39) + (1 << 26), 42)  # noqa: E731
for _ in range(3):
    c.native.agg_reset()
    run()
    c.native.agg_fetch()
torch.cuda.synchronize()
torch.cuda.profiler.start()
c.native.agg_reset()
run()
rc, bad, agg = c.native.agg_fetch()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
assert rc == 0, (rc, bad)
print("profiled one", what, "step:", agg.result()[1], "patchworks")
