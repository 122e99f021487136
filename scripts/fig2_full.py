"""Exhaustive 2^42 representative sweep of one degree-8 Fig-2 triangulation,
checkpointed per shard (long sweeps persist per-shard partial
reports; merge is associative, so a resumed run is identical).

    python scripts/fig2_full.py bowtie8 [--shards 64] [--out gpurun_out/fig2]

Writes <out>/<name>.ckpt.json after every shard and, at the end, the
reference-format report (<name>.jsonl, <name>.csv) plus a comparison with
the paper's published bins and distinct-scheme count.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2604_09221_b200 import Classifier, SweepRange, builtin, merge, sweep  # noqa: E402
from paper_2604_09221_b200.io import histogram_csv, report_jsonl  # noqa: E402
from paper_2604_09221_b200.sweep import SweepReport  # noqa: E402

# PAPER.md:916-1027 (percent of all 2^42 sign vectors per oval count) and :1036-1037
PUBLISHED = {
    "bowtie8": ({4: 4.6875, 6: 11.3281, 8: 14.6484, 10: 25.5371, 12: 17.1997, 14: 13.9526,
                 16: 10.9695, 18: 1.6113, 20: 0.0652, 22: 0.0004}, 123),
    "fig2-middle8": ({2: 0.2930, 3: 1.7578, 4: 4.1504, 5: 6.4941, 6: 10.0647, 7: 14.0991,
                      8: 15.6433, 9: 12.5443, 10: 6.7974, 11: 3.7655, 12: 4.5805, 13: 6.1824,
                      14: 6.3260, 15: 4.3626, 16: 2.0241, 17: 0.6985, 18: 0.1847, 19: 0.0253,
                      20: 0.0064}, 359),
    "fig2-right8": ({3: 0.0572, 4: 0.5581, 5: 2.5065, 6: 6.8969, 7: 13.0667, 8: 18.1908,
                     9: 19.4337, 10: 16.4603, 11: 11.3434, 12: 6.4880, 13: 3.1214, 14: 1.2716,
                     15: 0.4390, 16: 0.1279, 17: 0.0311, 18: 0.0062, 19: 0.0010, 20: 0.0001}, 353),
}


def to_json(r: SweepReport):
    return {"degree": r.degree, "fingerprint": r.fingerprint, "raw_space": r.raw_space,
            "hist": list(r.oval_histogram), "total": r.total_classified,
            "schemes": {s: list(v) for s, v in r.scheme_map.items()}}


def from_json(d):
    return SweepReport(d["degree"], d["fingerprint"], d["raw_space"], tuple(d["hist"]),
                       {s: tuple(v) for s, v in d["schemes"].items()}, d["total"])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("name")
    ap.add_argument("--shards", type=int, default=64)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "fig2"))
    args = ap.parse_args()
    os.makedirs(args.out, exist_ok=True)
    T = builtin(args.name)
    c = Classifier(T)
    domain = 1 << 42
    step = domain // args.shards
    ck = os.path.join(args.out, f"{args.name}.ckpt.json")
    done, acc, secs = 0, None, 0.0
    if os.path.exists(ck):
        with open(ck) as fh:
            st = json.load(fh)
        done, acc, secs = st["shards_done"], from_json(st["report"]), st["seconds"]
        print(f"resuming {args.name} at shard {done}/{args.shards}", flush=True)
    for s in range(done, args.shards):
        t0 = time.perf_counter()
        r = sweep(T, SweepRange(s * step, (s + 1) * step), classifier=c)
        secs += time.perf_counter() - t0
        acc = r if acc is None else merge(acc, r)
        with open(ck + ".tmp", "w") as fh:
            json.dump({"shards_done": s + 1, "seconds": secs, "report": to_json(acc)}, fh)
        os.replace(ck + ".tmp", ck)
        print(f"shard {s + 1}/{args.shards} {secs:.1f}s {acc.total_classified / secs:.3e}/s",
              flush=True)
    acc.params = {"mode": "sweep", "start": 0, "end": domain, "raw_space": False}
    with open(os.path.join(args.out, f"{args.name}.jsonl"), "w") as fh:
        fh.write(report_jsonl(acc))
    with open(os.path.join(args.out, f"{args.name}.csv"), "w") as fh:
        fh.write(histogram_csv(acc))
    bins, distinct = PUBLISHED[args.name]
    total = acc.total_classified
    cmp = {k: {"published_pct": v, "measured_pct": round(100.0 * acc.oval_histogram[k] / total, 4)}
           for k, v in bins.items()}
    extra = {k: c for k, c in enumerate(acc.oval_histogram) if c and k not in bins}
    summary = {"name": args.name, "total": total, "seconds": secs, "pps": total / secs,
               "distinct_schemes": acc.distinct_schemes(), "published_distinct": distinct,
               "bins": cmp, "mass_outside_published_bins": extra,
               "all_bins_match_4dp": all(abs(v["measured_pct"] - v["published_pct"]) < 5e-5
                                         for v in cmp.values())}
    with open(os.path.join(args.out, f"{args.name}.summary.json"), "w") as fh:
        json.dump(summary, fh, indent=1)
    print(json.dumps(summary), flush=True)


if __name__ == "__main__":
    main()
