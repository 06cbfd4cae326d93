"""Summarise an ncu report (kernels x key metrics) as a markdown table.
usage: python tools/ncu_summary.py report.ncu-rep [name-regex]"""
import csv
import re
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "dur"),
    ("smsp__inst_executed.sum", "inst"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64%"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu%"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma%"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1%"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "ld_conf"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "st_conf"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wf"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem%"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "st_long"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "st_short"),
    ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "st_mio"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "st_bar"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "st_wait"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "st_pipe"),
]


def main():
    rep = sys.argv[1]
    pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(m for m, _ in METRICS)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    print("| kernel | " + " | ".join(n for _, n in METRICS) + " |")
    print("|---" * (len(METRICS) + 1) + "|")
    for r in rows[2:]:
        d = dict(zip(h, r))
        name = re.sub(r"\(.*", "", d["Kernel Name"]).replace("(anonymous namespace)::", "")
        if pat and not pat.search(name):
            continue
        vals = []
        for m, _ in METRICS:
            v = d.get(m, "")
            try:
                f = float(v.replace(",", ""))
                vals.append(f"{f:.3g}" if f < 1e5 else f"{f / 1e3:.0f}K")
            except ValueError:
                vals.append(v or "-")
        print(f"| {name} | " + " | ".join(vals) + " |")
    print("\nunits: " + ", ".join(f"{n}={units[h.index(m)]}" for m, n in METRICS if m in h))


if __name__ == "__main__":
    main()
