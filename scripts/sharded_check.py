"""Two ranks (gloo) shard one sweep with distributed.sweep_sharded; the merged
report must equal a single-process sweep of the whole range."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2604_09221_b200 import SweepRange, builtin, sweep  # noqa: E402
from paper_2604_09221_b200.distributed import sweep_sharded  # noqa: E402

torch.cuda.set_device(0)
dist.init_process_group("gloo")
T = builtin("delaunay-7")
a, b = 123456789, 123456789 + (1 << 26) + 12345
rep = sweep_sharded(T, a, b, raw_space=True)
if dist.get_rank() == 0:
    ref = sweep(T, SweepRange(a, b), raw_space=True)
    ok = rep == ref and rep.total_classified == b - a
    print("sharded == single:", ok)
    assert ok
dist.destroy_process_group()
