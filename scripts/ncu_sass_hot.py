"""Per-instruction profile of an ncu capture: instructions executed per SASS
address, grouped into regions between branch targets; prints the hottest
instructions and the total.  Usage: python scripts/ncu_sass_hot.py rep [N]"""
import csv
import io
import subprocess
import sys


def main(path, top=60):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    data = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        try:
            n = int(r[ix["Instructions Executed"]] or 0)
        except ValueError:
            continue
        data.append((r[ix["Address"]], r[ix["Source"]], n, r[ix["Avg. Threads Executed"]],
                     r[ix["Warp Stall Sampling (All Samples)"]]))
    total = sum(d[2] for d in data)
    print(f"total warp instructions executed: {total:,}")
    ops = {}
    for a, s, n, t, w in data:
        op = s.split()[0] if s else "?"
        if op.startswith("@"):
            op = s.split()[1]
        op = op.split(".")[0]
        ops[op] = ops.get(op, 0) + n
    print("by opcode:", ", ".join(f"{k}:{v/total:.1%}" for k, v in sorted(ops.items(), key=lambda x: -x[1])[:25]))
    if top:
        for a, s, n, t, w in data:
            if n > total / 2000:
                print(f"{a} {n/total:7.3%} thr={t:>5} samp={w:>5}  {s}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 60)
