"""Write profiles/ncu_traffic.json from an ncu --set full capture: per kernel the
dram bytes per launch (read + write) and the issue / pipe counters bench.py
reports beside the roofline.  Usage:
  python scripts/ncu_to_json.py rep.ncu-rep "launch description" source-file"""
import csv
import io
import json
import subprocess
import sys

NAMES = {  # ncu kernel name prefix -> bench.py kernel label
    "k_tile_from_super": "k_tile_from_super",
    "k_super_build<4, 0>": "k_super_build<K=4,raw>",
    "k_tile_dedup": "k_tile_dedup",
    "k_l2_build": "k_l2_build",
    "k_l15_build": "k_l15_build",
    "k_l2_from_l15": "k_l2_from_l15 (+ k_l2_build)",
    "k_l2_dedup": "k_l2_dedup",
    "k_l2_classify": "k_l2_classify",
    "k_tile_classify<4, 0, 0>": "k_tile_classify<K=4,odd,raw>",
    "k_enumerate<4, 0, 0>": "k_enumerate<K=4,odd,raw>",
}


def main(path, launch, source):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    out = {}
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        name = d["Kernel Name"].replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
        name = name.replace("void ", "")
        label = next((v for k, v in NAMES.items() if name.startswith(k)), None)
        if label == "k_l2_dedup" and "k_l2_dedup (stage 1)" not in out:
            label = "k_l2_dedup (stage 1)"  # the first dedup of a step is stage 1's
        if label is None or label in out:
            continue
        f = lambda k: float(d[k].replace(",", "")) if d.get(k) else None  # noqa: E731
        rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
        # ncu reports Gbyte/Mbyte per the unit row; normalise to bytes
        units = dict(zip(hdr, rows[1]))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd *= scale.get(units["dram__bytes_read.sum"], 1)
        wr *= scale.get(units["dram__bytes_write.sum"], 1)
        out[label] = {
            "dram_bytes_per_launch": int(rd + wr), "dram_read": int(rd), "dram_write": int(wr),
            "time_ms_under_ncu": f("gpu__time_duration.sum") / (1e6 if units["gpu__time_duration.sum"] == "ns" else (1e3 if units["gpu__time_duration.sum"] == "us" else 1)),
            "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "alu_pipe_pct": f("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
            "threads_per_inst": f("smsp__thread_inst_executed_per_inst_executed.ratio"),
            "warps_active_pct": f("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "registers": f("launch__registers_per_thread"),
            "launch": launch, "source": source,
        }
    with open("profiles/ncu_traffic.json", "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:4])
