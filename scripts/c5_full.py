"""Config C5 at its stated scale: 10^12 uniform draws (seed 20260810) from a
degree-8 representative space on ONE B200, checkpointed per shard.

    python scripts/c5_full.py bowtie8 [--n 1000000000000] [--shard-log2 32]

The draws are the reference's counter sampler (kernels.py:439-462,
sweep.py:230-252): m_k = splitmix64(seed, k) & (2^42 - 1), k = 0..n-1, so
merging the shards equals ``sample(T, n, seed)`` (partition independence is
a GPU test).  At the end the oval histogram is compared with the published
Fig-2 bins (exhaustive percentages, so a 10^12-draw
sample must agree to ~1e-5 pp) and the report is written in the reference
formats.  SURVEY §0.1 quotes C5 as 10^12 draws across 8 GPUs.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2604_09221_b200 import Classifier, builtin, merge  # noqa: E402
from paper_2604_09221_b200.io import histogram_csv, report_jsonl  # noqa: E402
from paper_2604_09221_b200.sweep import SweepReport, sample_slice  # noqa: E402

PUBLISHED = {
    "bowtie8": {4: 4.6875, 6: 11.3281, 8: 14.6484, 10: 25.5371, 12: 17.1997, 14: 13.9526,
                16: 10.9695, 18: 1.6113, 20: 0.0652, 22: 0.0004},
    "fig2-middle8": {2: 0.2930, 3: 1.7578, 4: 4.1504, 5: 6.4941, 6: 10.0647, 7: 14.0991,
                     8: 15.6433, 9: 12.5443, 10: 6.7974, 11: 3.7655, 12: 4.5805, 13: 6.1824,
                     14: 6.3260, 15: 4.3626, 16: 2.0241, 17: 0.6985, 18: 0.1847, 19: 0.0253,
                     20: 0.0064},
}
SEED = 20260810


def to_json(r):
    return {"hist": list(r.oval_histogram), "total": r.total_classified,
            "schemes": {s: list(v) for s, v in r.scheme_map.items()},
            "degree": r.degree, "fingerprint": r.fingerprint}


def from_json(d):
    return SweepReport(d["degree"], d["fingerprint"], False, tuple(d["hist"]),
                       {s: tuple(v) for s, v in d["schemes"].items()}, d["total"])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("name")
    ap.add_argument("--n", type=int, default=10**12)
    ap.add_argument("--shard-log2", type=int, default=32)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "c5"))
    ap.add_argument("--budget-s", type=float, default=1e9, help="stop (resumable) after this")
    args = ap.parse_args()
    os.makedirs(args.out, exist_ok=True)
    T = builtin(args.name)
    c = Classifier(T)
    ck = os.path.join(args.out, f"{args.name}.ckpt.json")
    k0, acc, secs = 0, None, 0.0
    if os.path.exists(ck):
        with open(ck) as fh:
            st = json.load(fh)
        k0, acc, secs = st["next"], from_json(st["report"]), st["seconds"]
    step = 1 << args.shard_log2
    t_start = time.perf_counter()
    while k0 < args.n and time.perf_counter() - t_start < args.budget_s:
        k1 = min(args.n, k0 + step)
        t0 = time.perf_counter()
        r = sample_slice(T, SEED, k0, k1, classifier=c)
        secs += time.perf_counter() - t0
        acc = r if acc is None else merge(acc, r)
        k0 = k1
        with open(ck + ".tmp", "w") as fh:
            json.dump({"next": k0, "seconds": secs, "report": to_json(acc)}, fh)
        os.replace(ck + ".tmp", ck)
        print(f"{k0 / args.n:.4f} {secs:.0f}s {acc.total_classified / secs:.3e} draws/s",
              flush=True)
    if k0 < args.n:
        print("budget reached; resume with the same command", flush=True)
        return
    acc.params = {"mode": "sample", "n": args.n, "seed": SEED}
    with open(os.path.join(args.out, f"{args.name}.jsonl"), "w") as fh:
        fh.write(report_jsonl(acc))
    with open(os.path.join(args.out, f"{args.name}.csv"), "w") as fh:
        fh.write(histogram_csv(acc))
    pub = PUBLISHED.get(args.name, {})
    n = acc.total_classified
    bins = {k: {"published_pct": v, "sampled_pct": round(100.0 * acc.oval_histogram[k] / n, 6)}
            for k, v in pub.items()}
    summary = {"name": args.name, "draws": n, "seed": SEED, "seconds": secs,
               "draws_per_s": n / secs, "distinct_schemes": acc.distinct_schemes(),
               "bins": bins,
               "max_abs_diff_pp": max((abs(b["sampled_pct"] - b["published_pct"])
                                       for b in bins.values()), default=None)}
    with open(os.path.join(args.out, f"{args.name}.summary.json"), "w") as fh:
        json.dump(summary, fh, indent=1)
    print(json.dumps(summary), flush=True)


if __name__ == "__main__":
    main()
