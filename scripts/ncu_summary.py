"""Key metrics + stall breakdown per kernel of an .ncu-rep (read here with ncu -i)."""
import csv, io, subprocess, sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__grid_size",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__thread_inst_executed_per_inst_executed.ratio"]


def summary(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        out.append(f"== {r[h.index('Kernel Name')] if 'Kernel Name' in h else r[4]}")
        for i, n in enumerate(h):
            if n in WANT:
                out.append(f"  {n:65s} {r[i]:>16s} {u[i]}")
        st = []
        for i, n in enumerate(h):
            if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
                try:
                    st.append((float(r[i]), n[34:-23]))
                except ValueError:
                    pass
        out.append("  stalls per issued instruction: " + ", ".join(f"{b} {a:.2f}" for a, b in sorted(st, reverse=True)[:7]))
    return "\n".join(out)


if __name__ == "__main__":
    print(summary(sys.argv[1]))
