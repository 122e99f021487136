"""Generate tests/golden/c3_full.json: the complete C3 report (delaunay-7, raw
lower half [0, 2^35) = the full 2^36 space mod the global sign flip) from the
pinned CPU oracle, as 32 pieces of 2^30 indices.

TEST INFRASTRUCTURE ONLY.  The oracle (oracle/tcg_oracle.c) is itself pinned
to reference-produced fixtures by tests/test_oracle.py; this script only runs
it over the whole headline domain (about 5 CPU-hours on 8 threads), once, in
the build container.  Resumable: finished pieces are kept in the output file.

Each piece is the reference's sweep report restricted to that index range
(sweep.py:198-227 with raw_space=True): histogram, scheme -> (count, smallest
raw index), total.  The GPU tests merge pieces (count sum, witness min,
sweep.py:83-105) to get the two bench chunks [0,2^34), [2^34,2^35) and the
whole domain.

    python tests/golden/make_c3_full.py [threads]
"""

from __future__ import annotations

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2604_09221_b200 import builtin  # noqa: E402
from paper_2604_09221_b200.diamond import plan_arrays, reflect  # noqa: E402

OUT = os.path.join(HERE, "c3_full.json")
PIECE_LOG2 = 30
NPIECES = 32


def main() -> None:
    threads = int(sys.argv[1]) if len(sys.argv) > 1 else os.cpu_count()
    T = builtin("delaunay-7")
    plan = O.OraclePlan.from_arrays(plan_arrays(reflect(T)))
    doc = {"triangulation": "delaunay-7", "raw_space": True, "piece_log2": PIECE_LOG2,
           "generator": "oracle/tcg_oracle.c orc_sweep (pinned by tests/test_oracle.py)",
           "pieces": {}}
    if os.path.exists(OUT):
        with open(OUT) as f:
            doc = json.load(f)
    for p in range(NPIECES):
        if str(p) in doc["pieces"]:
            continue
        a, b = p << PIECE_LOG2, (p + 1) << PIECE_LOG2
        t0 = time.time()
        r = O.sweep(plan, True, a, b, threads=threads, chunk=1 << 18)
        assert r["status"] == 0, r["status"]
        M = 16
        assert all(x == 0 for x in r["hist"][M + 1:])
        doc["pieces"][str(p)] = {
            "start": a, "end": b, "total": r["total"], "hist": r["hist"][: M + 1],
            "schemes": {s: list(cw) for s, cw in sorted(r["schemes"].items())},
            "cpu_s": round(time.time() - t0, 1),
        }
        tmp = OUT + ".tmp"
        with open(tmp, "w") as f:
            json.dump(doc, f, sort_keys=True, separators=(",", ":"))
        os.replace(tmp, OUT)
        print(f"piece {p}: [{a}, {b}) {len(r['schemes'])} schemes in {time.time() - t0:.0f} s",
              flush=True)


if __name__ == "__main__":
    main()
