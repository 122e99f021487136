"""Determinism stress of the any-degree kernel (k_large) on the inputs of
tests/test_gpu_parity.py::test_acceptance_criterion_10_degree_scaling:
classify every row many times and report statuses / disagreements."""
import random
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2604_09221_b200 import Classifier, lattice_points, num_points  # noqa: E402
from paper_2604_09221_b200.lifting import from_lifting  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
rng = random.Random(0x5CA1E)
for d, calls in ((24, 60), (48, 30)):
    T = None
    while T is None or not T.is_unimodular:
        lift = {(i, j): 8 * (i * i + i * j + j * j) + rng.randint(0, 1) for i, j in lattice_points(d)}
        T = from_lifting(d, lift)
    c = Classifier(T, device=0)
    batches = [np.array([rng.randint(0, 1) for _ in range(num_points(d))], np.uint8)
               for _ in range(calls)]
    words = (num_points(d) + 63) // 64
    rows = np.zeros((len(batches), words), np.uint64)
    for t, bits in enumerate(batches):
        b = np.asarray(bits, dtype=np.uint64)
        for w in range(words):
            ch = b[64 * w: 64 * w + 64]
            rows[t, w] = np.bitwise_or.reduce(ch << np.arange(len(ch), dtype=np.uint64))
    ref = None
    bad = 0
    for r in range(reps):
        for t in range(len(rows)):
            st, nr, par = c.large.classify_rows(rows[t:t + 1])
            key = (int(st[0]), int(nr[0]), tuple(int(x) for x in par[0][:int(nr[0])]))
            if r == 0:
                ref = ref or {}
                ref[t] = key
            elif key != ref[t]:
                bad += 1
                if bad < 10:
                    print(f"d={d} row {t} rep {r}: {key[:2]} vs {ref[t][:2]}", flush=True)
        st, nr, par = c.large.classify_rows(rows)  # whole batch at once
        for t in range(len(rows)):
            key = (int(st[t]), int(nr[t]), tuple(int(x) for x in par[t][:int(nr[t])]))
            if key != ref[t]:
                bad += 1
                if bad < 10:
                    print(f"d={d} row {t} batch rep {r}: {key[:2]} vs {ref[t][:2]}", flush=True)
    nonok = sum(1 for k in ref.values() if k[0] != 0)
    print(f"d={d}: {len(rows)} rows x {reps} reps, first-pass non-OK {nonok}, disagreements {bad}", flush=True)
