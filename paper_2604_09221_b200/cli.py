"""Command line for the classification path.

Same subcommands, flags, output lines and exit codes as the reference CLI
for the path (reference cli.py:55-109, 191-282): ``classify``, ``sweep``,
``sample``, ``export-builtin``; plus ``batch`` (many sign vectors for one
triangulation in one launch).  Exit codes: 0 ok, 2 malformed input (or no
usable GPU), 3 violated invariant, 4 budget exceeded.  Reports are written
with the reference's byte format (io.py), so files are interchangeable.

    python -m paper_2604_09221_b200 sweep --builtin delaunay-7 --raw-sign-space \\
        --output r.jsonl --histogram h.csv
"""

from __future__ import annotations

import argparse
import json
import sys
import time

from .builtins import builtin
from .classify import Classifier
from .errors import BudgetExceeded, InvariantViolation, ParseError, TcurvesError
from .io import read_signs, read_triangulation, write_report, write_triangulation
from .sweep import SweepRange, sample, sweep


def _triangulation(args):
    if (args.triangulation is None) == (args.builtin is None):
        raise ParseError("provide a triangulation file or --builtin, not both")
    if args.builtin:
        return builtin(args.builtin)
    return read_triangulation(args.triangulation, require_unimodular=not args.skip_validation)


def _summary(report, elapsed):
    rate = report.total_classified / elapsed if elapsed > 0 else float("inf")
    print(f"classified: {report.total_classified}")
    print(f"distinct schemes: {report.distinct_schemes()}")
    print(f"max ovals: {report.max_ovals()}")
    print(f"wall time: {elapsed:.2f} s ({rate:,.0f}/s)")


def cmd_classify(args):
    T = _triangulation(args)
    res = Classifier(T, device=args.device).classify(read_signs(T.degree, args.signs))
    if args.json:
        print(json.dumps(res.to_dict(), sort_keys=True))
    else:
        print(res.scheme)
        print(f"ovals: {res.oval_count}")
        print(f"pseudoline: {'yes' if res.has_pseudoline else 'no'}")
    return 0


def cmd_batch(args):
    T = _triangulation(args)
    with open(args.signs_file) as fh:
        lines = [ln.strip() for ln in fh if ln.strip()]
    res = Classifier(T, device=args.device).classify_many(lines)
    for s, r in zip(lines, res):
        if args.json:
            print(json.dumps({"signs": s, **r.to_dict()}, sort_keys=True))
        else:
            print(f"{s} {r.scheme}")
    return 0


def cmd_sweep(args):
    T = _triangulation(args)
    rng = None
    if args.start is not None or args.end is not None:
        if args.start is None or args.end is None:
            raise ParseError("--start and --end must be given together")
        rng = SweepRange(args.start, args.end)
    devices = [int(x) for x in args.devices.split(",")] if args.devices else None
    t0 = time.perf_counter()
    report = sweep(T, rng, workers=args.workers, raw_space=args.raw_sign_space,
                   chunk_size=args.chunk_size, devices=devices)
    elapsed = time.perf_counter() - t0
    write_report(report, args.output, args.histogram)
    _summary(report, elapsed)
    return 0


def cmd_sample(args):
    T = _triangulation(args)
    devices = [int(x) for x in args.devices.split(",")] if args.devices else None
    t0 = time.perf_counter()
    report = sample(T, args.n, args.seed, workers=args.workers, chunk_size=args.chunk_size,
                    devices=devices)
    elapsed = time.perf_counter() - t0
    write_report(report, args.output, args.histogram)
    _summary(report, elapsed)
    return 0


def cmd_export_builtin(args):
    write_triangulation(builtin(args.name), args.output)
    print(args.output)
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_2604_09221_b200",
                                 description="B200 real-scheme classifier for patchworks")
    sub = ap.add_subparsers(dest="command", required=True)

    def inputs(p):
        p.add_argument("triangulation", nargs="?", help="triangulation JSON file")
        p.add_argument("--builtin", help="use a builtin triangulation instead of a file")
        p.add_argument("--skip-validation", action="store_true",
                       help="do not require unimodularity")
        p.add_argument("--device", type=int, default=None, help="CUDA device (default: current)")

    def reports(p):
        p.add_argument("--workers", type=int, default=1, help="accepted; results never depend on it")
        p.add_argument("--chunk-size", type=int, default=1 << 16)
        p.add_argument("--devices", help="comma-separated GPU ids to shard over (one process)")
        p.add_argument("--output", help="JSONL scheme report path")
        p.add_argument("--histogram", help="CSV oval histogram path")

    p = sub.add_parser("classify", help="print the real scheme of one patchwork")
    inputs(p)
    p.add_argument("signs", help="sign bitstring in canonical point order")
    p.add_argument("--json", action="store_true")
    p.set_defaults(fn=cmd_classify)

    p = sub.add_parser("batch", help="classify every sign bitstring of a file (one per line)")
    inputs(p)
    p.add_argument("signs_file")
    p.add_argument("--json", action="store_true")
    p.set_defaults(fn=cmd_batch)

    p = sub.add_parser("sweep", help="classify a range of sign indices")
    inputs(p)
    p.add_argument("--start", type=int)
    p.add_argument("--end", type=int)
    p.add_argument("--raw-sign-space", action="store_true")
    reports(p)
    p.set_defaults(fn=cmd_sweep)

    p = sub.add_parser("sample", help="classify seeded uniform sign draws")
    inputs(p)
    p.add_argument("-n", type=int, required=True)
    p.add_argument("--seed", type=int, default=0)
    reports(p)
    p.set_defaults(fn=cmd_sample)

    p = sub.add_parser("export-builtin", help="write a builtin triangulation to JSON")
    p.add_argument("name")
    p.add_argument("output")
    p.set_defaults(fn=cmd_export_builtin)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.fn(args)
    except InvariantViolation as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 3
    except BudgetExceeded as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 4
    except (TcurvesError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
