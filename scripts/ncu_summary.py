#!/usr/bin/env python3
"""Summarise an ncu --set full report: key throughput metrics + top stall reasons per kernel."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__bytes.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "lts__t_sector_hit_rate.pct",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units, data = rows[0], rows[1], rows[2:]
    ki = h.index("Kernel Name")
    for r in data:
        print("=" * 100)
        print(r[ki][:100])
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"  {k:65s} {r[i]:>16s} {units[i]}")
        st = [(h[i], r[i]) for i in range(len(h)) if h[i].startswith("smsp__pcsamp_warps_issue_stalled")
              and not h[i].endswith("not_issued")]

        def f(x):
            try:
                return float(x.replace(",", ""))
            except ValueError:
                return 0.0
        st.sort(key=lambda x: -f(x[1]))
        tot = sum(f(v) for _, v in st) or 1
        print("  stalls: " + ", ".join(f"{k.split('stalled_')[1]} {100 * f(v) / tot:.0f}%"
                                        for k, v in st[:7]))


if __name__ == "__main__":
    main(sys.argv[1])
