"""Small profiling target: a few sweeps / samples of one builtin (for ncu).
python scripts/prof_target.py bowtie8 rep 0x4000000000 0x4000000 [sample]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_09221_b200 import Classifier, SweepRange, builtin, sweep  # noqa: E402
from paper_2604_09221_b200.sweep import sample_slice  # noqa: E402

name, dom, a, n = sys.argv[1], sys.argv[2], int(sys.argv[3], 0), int(sys.argv[4], 0)
T = builtin(name)
c = Classifier(T)
for rep in range(3):
    if dom == "sample":
        r = sample_slice(T, 20260810, a, a + n, classifier=c)
    else:
        r = sweep(T, SweepRange(a, a + n), raw_space=dom == "raw", classifier=c)
print(r.total_classified, r.distinct_schemes())
