"""Time the phases of one C4 e2e step (MultiClassifier.classify_words, 2^28 pairs)."""
import os
import sys
import time

sys.path.insert(0, ".")
os.environ.setdefault("TCG_HOST_TRACE", "1")
import numpy as np  # noqa: E402

from paper_2604_09221_b200 import MultiClassifier  # noqa: E402
from paper_2604_09221_b200.lattice import Triangulation  # noqa: E402

data = np.load("tests/golden/c4_d7_4096.npz")
Ts = [Triangulation(7, tuple(((int(a), int(b)), (int(c), int(d))) for a, b, c, d in e), ())
      for e in data["edges"].astype(int)]
mc = MultiClassifier(Ts, device=0)
n, per = 1 << 28, 1 << 16
k = np.arange(n, dtype=np.uint64)
z = np.uint64(7) + (k + np.uint64(1)) * np.uint64(0x9E3779B97F4A7C15)
z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
words = (z ^ (z >> np.uint64(31))) & np.uint64((1 << 36) - 1)
tri = (np.arange(n, dtype=np.int64) // per).astype(np.int32)
for i in range(3):
    t0 = time.perf_counter()
    r = mc.classify_words(tri, words)
    print(f"call {i}: {time.perf_counter() - t0:.3f} s  kernel {mc.native.last_ms():.1f} ms", flush=True)
