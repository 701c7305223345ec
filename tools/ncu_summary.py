"""Summarise an ncu raw CSV (one kernel) + source CSV hot spots."""
import csv, sys
def raw(path):
    rows = list(csv.reader(open(path)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    return {h: (data[0][i], units[i]) for i, h in enumerate(hdr)} if data else {}
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg", "smsp__cycles_active.avg",
        "smsp__inst_executed.sum", "launch__grid_size", "launch__registers_per_thread",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio",
        "smsp__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__warps_active.avg.per_cycle_active", "smsp__cycles_elapsed.avg.per_second"]
def main(prefix):
    r = raw(prefix + ".raw.csv")
    for k in KEYS:
        if k in r: print("%-85s %s %s" % (k, r[k][0], r[k][1]))
    rows = list(csv.reader(open(prefix + ".source.csv")))
    hdr = rows[1] if rows[0] and rows[0][0] == "Kernel Name" else rows[0]
    data = rows[2:] if rows[0] and rows[0][0] == "Kernel Name" else rows[1:]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    tot = sum(int(x[si]) for x in data if len(x) > si and x[si].isdigit())
    print("stall samples", tot)
    for x in sorted((x for x in data if len(x) > si and x[si].isdigit()), key=lambda x: -int(x[si]))[:12]:
        print("  %5s %s" % (x[si], x[1][:90]))
if __name__ == "__main__":
    main(sys.argv[1])
