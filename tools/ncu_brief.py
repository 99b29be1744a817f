#!/usr/bin/env python3
"""One-screen summary of an ncu --set full report: time, issue/pipe use,
occupancy, stall reasons per issue, DRAM traffic.
usage: python tools/ncu_brief.py report.ncu-rep [...]"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum"]
for path in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        print(f"== {path}: {v[h.index('Kernel Name')][:90]}")
        for a, b, c in zip(h, u, v):
            if a in KEYS:
                print(f"  {a:60s} {c:>14s} {b}")
        st = [(a.split("stalled_")[1].replace("_per_issue_active.ratio", ""), float(c))
              for a, c in zip(h, v)
              if a.startswith("smsp__average_warps_issue_stalled_") and a.endswith("per_issue_active.ratio")
              and c not in ("", "n/a")]
        st.sort(key=lambda t: -t[1])
        print("  stalls/issue: " + ", ".join(f"{k} {x:.2f}" for k, x in st[:8]))
