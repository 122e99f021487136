"""Summarise an ncu --set full capture (run here, on the CPU box): the
counters the design is judged by (issue, ALU pipe, divergence, spills,
DRAM bytes, stall reasons).  Usage: python scripts/ncu_summary.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.avg.per_cycle_active", "sm__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.sum", "sm__inst_executed_pipe_lsu.sum",
    "sm__inst_executed_pipe_uniform.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        d, u = dict(zip(hdr, vals)), dict(zip(hdr, units))
        for k in KEYS:
            if k in d:
                print(f"{k:70s} {d[k]} {u.get(k, '')}")
        st = [(k, d[k]) for k in hdr if k.startswith("smsp__average_warps_issue_stalled_")
              and k.endswith("_per_issue_active.ratio")]
        st = sorted(st, key=lambda x: -float(x[1] or 0))[:10]
        print("top stall reasons (warps per issue-active cycle):")
        for k, v in st:
            print(f"  {k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]:30s} {v}")


if __name__ == "__main__":
    main(sys.argv[1])
