"""Summarise an ncu report: key raw metrics + stall reasons + hottest SASS lines.

    python tools/ncu_summary.py report.ncu-rep [--lines N]
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__occupancy_limit_registers",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct", "launch__shared_mem_per_block_dynamic",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed_op_shared_st.sum",
        "smsp__inst_executed_op_shared_ld.sum", "smsp__inst_executed_op_global_ld.sum",
        "smsp__inst_executed_op_global_st.sum"]


def ncu(path, *args):
    return subprocess.run(["ncu", "-i", path, *args], capture_output=True, text=True).stdout


def main():
    path = sys.argv[1]
    nlines = int(sys.argv[sys.argv.index("--lines") + 1]) if "--lines" in sys.argv else 25
    rows = list(csv.reader(io.StringIO(ncu(path, "--page", "raw", "--csv"))))
    h, units, r = rows[0], rows[1], rows[2]
    print("kernel:", r[h.index("Kernel Name")][:120])
    for k in KEYS:
        if k in h:
            print(f"  {k:70s} {r[h.index(k)]} {units[h.index(k)]}")
    stalls = []
    for i, k in enumerate(h):
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(r[i]), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    print("  stalls per issue:", ", ".join(f"{n}={v:.2f}" for v, n in sorted(stalls, reverse=True)[:8]))
    src = list(csv.reader(io.StringIO(ncu(path, "--page", "source", "--csv", "--print-source", "sass"))))
    hh = src[1]
    ie, st, sa = hh.index("Instructions Executed"), hh.index("Warp Stall Sampling (All Samples)"), hh.index("Source")
    data = src[2:]
    tot_i = sum(int(x[ie] or 0) for x in data)
    tot_s = sum(int(x[st] or 0) for x in data)
    print(f"  warp instructions {tot_i}, stall samples {tot_s}")
    hot = sorted(range(len(data)), key=lambda i: -int(data[i][st] or 0))[:nlines]
    for i in sorted(hot):
        print(f"  {i:5d} inst={data[i][ie]:>9s} samples={data[i][st]:>5s}  {data[i][sa].strip()[:80]}")


if __name__ == "__main__":
    main()
