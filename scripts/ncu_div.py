"""Warp instructions and active threads per CUDA source line (divergence map).
Usage: python scripts/ncu_div.py rep.ncu-rep kernel-regex [top]"""
import csv
import io
import subprocess
import sys


def main(path, kregex, top=30):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source",
                          "sass,cuda", "-k", f"regex:{kregex}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    fname, hdr, per = "?", None, []
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0].isdigit():
            continue
        try:
            wi = float(r[hdr.index("Instructions Executed")] or 0)
            ti = float(r[hdr.index("Thread Instructions Executed")] or 0)
        except (ValueError, IndexError):
            continue
        if wi:
            per.append((wi, ti, fname, int(r[0]), r[1].strip()[:70]))
    W = sum(p[0] for p in per)
    T = sum(p[1] for p in per)
    print(f"warp inst {W:.3e}  thread inst {T:.3e}  threads/inst {T / W:.2f}")
    print("lost lane-slots by line (32*warp_inst - thread_inst):")
    per.sort(key=lambda p: -(32 * p[0] - p[1]))
    for wi, ti, f, ln, src in per[:top]:
        print(f"{f:10s} {ln:5d} {100 * wi / W:5.1f}% inst  {ti / wi:5.1f} thr  lost {100 * (32 * wi - ti) / (32 * W - T):5.1f}%  {src}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30)
