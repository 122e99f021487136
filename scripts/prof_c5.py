"""C5 sampling launch for profiling: 2^24 draws at k0 = 2^39 (default bowtie8).
The first slice builds the split tables (k_split_build) and warms the
sampler; profile the second k_sample_split launch (ncu -k regex:k_sample -s 1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_09221_b200 import Classifier, builtin  # noqa: E402
from paper_2604_09221_b200.sweep import sample_slice  # noqa: E402

T = builtin(sys.argv[1] if len(sys.argv) > 1 else "bowtie8")
c = Classifier(T)
c.native.set_split(True)  # the split path from the first slice on
sample_slice(T, 20260810, 0, 1 << 20, classifier=c)
r = sample_slice(T, 20260810, 1 << 39, (1 << 39) + (1 << 24), classifier=c)
print(r.total_classified, c.native.split_stats())
