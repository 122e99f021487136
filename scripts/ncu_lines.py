"""Instructions executed and stall samples per CUDA source line (needs -lineinfo).
Usage: python scripts/ncu_lines.py rep.ncu-rep kernel-regex [top]"""
import csv
import io
import subprocess
import sys


def main(path, kregex, top=40):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source",
                          "sass,cuda", "-k", f"regex:{kregex}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    per = {}
    cur = None
    total = 0
    fname = "?"
    iexe = isamp = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            iexe = r.index("Instructions Executed")
            isamp = r.index("Warp Stall Sampling (All Samples)")
            continue
        if iexe is None or len(r) <= iexe:
            continue
        if r[0].isdigit():
            cur = (fname, int(r[0]), r[1].strip()[:70])
            continue
        if not r[2].startswith("0x"):
            continue
        try:
            n = int(r[iexe] or 0)
            s = int(r[isamp] or 0)
        except ValueError:
            continue
        if cur:
            e = per.setdefault(cur, [0, 0])
            e[0] += n
            e[1] += s
        total += n
    print(f"total instructions {total:,}")
    tops = sorted(per.items(), key=lambda x: -x[1][0])[:top]
    for (fn, ln, src), (n, s) in sorted(tops):
        print(f"{fn[:10]:10s} {ln:5d} {100.0 * n / total:6.2f}%  samp {s:7d}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
