"""Summarise an ncu report (details page) into a small table.

  python tools/ncu_summary.py gpurun_out/prof.ncu-rep [> profiles/xxx.txt]
"""
import csv
import io
import subprocess
import sys

WANT = ("Duration", "DRAM Throughput", "Memory Throughput", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "Compute (SM) Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Warp Cycles Per Issued Instruction",
        "Executed Ipc Active", "Block Limit Shared Mem", "Block Limit Registers",
        "Dynamic Shared Memory Per Block", "Grid Size", "Block Size", "Waves Per SM",
        "Issue Slots Busy", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Avg. Active Threads Per Warp", "Avg. Not Predicated Off Threads Per Warp",
        "Branch Efficiency", "SM Frequency", "DRAM Frequency")
RAW = ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
       "smsp__thread_inst_executed_per_inst_executed.ratio",
       "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
       "sm__inst_executed_pipe_fp64.sum", "sm__inst_executed_pipe_alu.sum",
       "smsp__average_warp_latency_issue_stalled_long_scoreboard",
       "dram__throughput.avg.pct_of_peak_sustained_elapsed",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active")


def main(path):
    det = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    r = csv.reader(io.StringIO(det))
    h = next(r)
    ki, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value",
                                          "Metric Unit"))
    ii = h.index("ID")
    rows = {}
    for row in r:
        if row[mi] in WANT:
            rows.setdefault((row[ii], row[ki][:60]), []).append(f"{row[mi]} = {row[vi]} {row[ui]}")
    for (i, k), ms in rows.items():
        print(f"== launch {i}: {k}")
        for m in ms:
            print("   ", m)
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    if len(r) > 2:
        h = r[0]
        units = r[1]
        for row in r[2:]:
            name = row[h.index("Kernel Name")][:60]
            print(f"== raw: {name}")
            for m in RAW:
                if m in h:
                    j = h.index(m)
                    print(f"    {m} = {row[j]} {units[j]}")


if __name__ == "__main__":
    main(sys.argv[1])
