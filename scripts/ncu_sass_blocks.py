"""Instruction counts per basic block (runs of equal execution count) of an
ncu capture, to see where a kernel's instructions go.
Usage: python scripts/ncu_sass_blocks.py rep.ncu-rep [min_pct]"""
import csv
import io
import subprocess
import sys


def main(path, min_pct=0.5):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    sections, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = [r[1], None, []]
            sections.append(cur)
        elif cur is not None and cur[1] is None:
            cur[1] = r
        elif cur is not None:
            cur[2].append(r)
    for name, hdr, body in sections:
        print("==", name[:100])
        report(hdr, body, min_pct)


def report(hdr, body, min_pct):
    ix = {h: i for i, h in enumerate(hdr)}
    data = []
    for r in body:
        if len(r) != len(hdr):
            continue
        try:
            n = int(r[ix["Instructions Executed"]] or 0)
        except ValueError:
            continue
        data.append((r[ix["Address"]], r[ix["Source"]], n))
    total = sum(d[2] for d in data)
    blocks = []
    for a, s, n in data:
        if blocks and blocks[-1][2] == n:
            blocks[-1][1] += 1
            blocks[-1][3].append(s)
        else:
            blocks.append([a, 1, n, [s]])
    print(f"total {total:,}")
    for a, ln, n, srcs in blocks:
        pct = 100.0 * ln * n / total
        if pct >= min_pct:
            ops = {}
            for s in srcs:
                op = s.split()[1] if s.startswith("@") else s.split()[0]
                op = op.split(".")[0]
                ops[op] = ops.get(op, 0) + 1
            top = " ".join(f"{k}{v}" for k, v in sorted(ops.items(), key=lambda x: -x[1])[:6])
            print(f"{a[-5:]} len {ln:4d} execs {n:>12,} {pct:6.2f}%  {top}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 0.5)
