"""profiles/ncu_kernels.json from an ncu --set full capture of ONE bench step
(scripts/profile_step.py): per kernel, sums over the step's launches of
thread instructions, dram bytes and time, plus launch-weighted utilisation
counters; tagged with the sha of the tcg.cu it was built from (bench.py
uses the file only when the sha matches the source it runs).

    python scripts/ncu_kernels_json.py rep.ncu-rep out.json "description"
"""
import csv
import hashlib
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6,
         "inst": 1, "Kinst": 1e3, "Minst": 1e6, "Ginst": 1e9, "sector": 1, "Ksector": 1e3,
         "Msector": 1e6, "Gsector": 1e9}


def short(name):
    name = name.replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    name = name.replace("void ", "")
    return name.split("<")[0].split("(")[0]


def main(path, out_path, desc):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], dict(zip(rows[0], rows[1]))

    def val(d, k):
        v = d.get(k)
        if v in (None, "", "n/a"):
            return None
        return float(v.replace(",", "")) * SCALE.get(units.get(k, ""), 1)

    acc = {}
    prev = None
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        name = short(d["Kernel Name"])
        if name == "k_l2_dedup":
            name += "/stage1" if prev == "k_l15_build" else "/level2"
        else:
            prev = name
        a = acc.setdefault(name, {"launches": 0, "thread_inst_per_step": 0.0,
                                  "inst_per_step": 0.0, "dram_bytes_per_step": 0.0,
                                  "ncu_time_ns_per_step": 0.0, "local_sectors_per_step": 0.0,
                                  "_w": {}})
        a["launches"] += 1
        t = val(d, "gpu__time_duration.sum") or 0.0
        a["ncu_time_ns_per_step"] += t
        a["thread_inst_per_step"] += val(d, "smsp__thread_inst_executed.sum") or 0.0
        a["inst_per_step"] += val(d, "smsp__inst_executed.sum") or 0.0
        a["dram_bytes_per_step"] += ((val(d, "dram__bytes_read.sum") or 0.0) +
                                     (val(d, "dram__bytes_write.sum") or 0.0))
        a["local_sectors_per_step"] += ((val(d, "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum") or 0)
                                        + (val(d, "l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum") or 0))
        for k, lab in (("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
                       ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu_pipe_pct"),
                       ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads_per_inst"),
                       ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
                       ("launch__registers_per_thread", "registers"),
                       ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct_of_peak")):
            v = val(d, k)
            if v is not None:
                w = a["_w"].setdefault(lab, [0.0, 0.0])
                w[0] += v * t
                w[1] += t
    for a in acc.values():
        for lab, (s, t) in a.pop("_w").items():
            a[lab] = round(s / t, 3) if t else None
    d = os.path.join(ROOT, "paper_2604_09221_b200", "csrc")
    h = hashlib.sha256()
    for f in sorted(os.listdir(d)):  # same digest as bench.py source_sha16
        if f.endswith((".cu", ".cuh")):
            with open(os.path.join(d, f), "rb") as fh:
                h.update(fh.read())
    sha = h.hexdigest()[:16]
    doc = {"tcg_cu_sha16": sha, "capture": desc, "report": os.path.basename(path),
           "kernels": acc}
    with open(out_path, "w") as fh:
        json.dump(doc, fh, indent=1, sort_keys=True)
    print(json.dumps(doc, indent=1, sort_keys=True))


if __name__ == "__main__":
    main(*sys.argv[1:4])
