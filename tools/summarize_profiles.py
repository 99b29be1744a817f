#!/usr/bin/env python3
"""Turns the round's ncu outputs (gpurun_out/) into tracked summaries under
profiles/: per-program DRAM traffic per launch (the bench's roofline
`traffic`), the bench launch list aggregated per kernel, and the key
metrics of the full captures.

usage: python tools/summarize_profiles.py <round tag, e.g. r01>
"""
import collections
import csv
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GO = os.path.join(ROOT, "gpurun_out")
PR = os.path.join(ROOT, "profiles")
PROGRAMS = [f"{w}/{s}" for w in ("cdf53", "cdf97") for s in (
    "sweldens", "iwahashi", "iwahashi_star", "explosive", "explosive_star", "monolithic",
    "monolithic_star", "polyphase", "polyphase_star", "convolution")]


def read_metrics_csv(path):
    """[(kernel name, {metric: (value, unit)})] in launch order."""
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi, ui, ii = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                          h.index("Metric Unit"), h.index("ID"))
    launches = collections.OrderedDict()
    for r in rows[hi + 1:]:
        d = launches.setdefault(r[ii], (r[ki], {}))
        d[1][r[mi]] = (float(r[vi].replace(",", "")), r[ui])
    return list(launches.values())


def to_bytes(v, u):
    return v * {"byte": 1, "Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6, "Gbyte": 1e9, "GB": 1e9}.get(u, 1)


def to_us(v, u):
    return v * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}.get(u, 1)


def short(name):
    m = re.search(r"P_(cdf\d+)_(\w+?)_(fwd|inv)", name)
    if m:
        return f"fast {m.group(1)}/{m.group(2)}/{m.group(3)}"
    m = re.search(r"conv_fast_kernel<Conv_(cdf\d+)>", name)
    if m:
        return f"conv {m.group(1)}/convolution/fwd"
    return re.sub(r"\(.*", "", name).replace("void ", "").replace("(anonymous namespace)::", "")


def main(tag):
    os.makedirs(PR, exist_ok=True)
    # 1. traffic per launch: tools/bench_kernels.py 8192 1 <20 programs> ->
    #    8 launches per program (3 warm-up fwd/inv pairs + 1 timed pair)
    tr = read_metrics_csv(os.path.join(GO, f"traffic_{tag}.csv"))
    kern = [k for k in tr if "uniform_kernel" not in k[0] and "elementwise" not in k[0]]
    traffic = {}
    for i, p in enumerate(PROGRAMS):
        pair = kern[8 * i + 6: 8 * i + 8]
        for d, (name, m) in zip(("fwd", "inv"), pair):
            rb = to_bytes(*m["dram__bytes_read.sum"])
            wb = to_bytes(*m["dram__bytes_write.sum"])
            traffic[f"{p}/{d}"] = {"read": rb, "write": wb, "total": rb + wb,
                                   "algorithmic": 8.0 * 8192 * 8192,
                                   "us": to_us(*m["gpu__time_duration.sum"]),
                                   "kernel": short(name)}
    json.dump({k: v["total"] for k, v in traffic.items()},
              open(os.path.join(PR, f"traffic_{tag}.json"), "w"), indent=1)
    # 2. launch list of the bench command, aggregated per kernel
    ll = read_metrics_csv(os.path.join(GO, f"launches_{tag}.csv"))
    agg = collections.defaultdict(list)
    for name, m in ll:
        agg[short(name)].append(to_us(*m["gpu__time_duration.sum"]))
    tot = sum(sum(v) for v in agg.values())
    lines = [f"# ncu launch list, round {tag}",
             "",
             "`ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv "
             "python bench.py --steps 1 --warmup 1 --no-c3 --no-c4 --no-c5 --e2e-steps 0 --no-cpu` (raw: "
             f"`launches_{tag}.csv`). Cold-cache, serialised: compare shares, not absolutes.",
             "", "| kernel | launches | mean us | share of listed time |", "|---|---:|---:|---:|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| {k} | {len(v)} | {sum(v) / len(v):.1f} | {sum(v) / tot:.3f} |")
    lines += ["", f"## DRAM traffic per launch at 8192^2 (`traffic_{tag}.csv`)", "",
              "| program | kernel | read GB | write GB | total / algorithmic | us |",
              "|---|---|---:|---:|---:|---:|"]
    for p, v in traffic.items():
        lines.append(f"| {p} | {v['kernel']} | {v['read'] / 1e9:.3f} | {v['write'] / 1e9:.3f} | "
                     f"{v['total'] / v['algorithmic']:.3f} | {v['us']:.1f} |")
    open(os.path.join(PR, f"launches_{tag}.md"), "w").write("\n".join(lines) + "\n")
    # 3. full captures -> raw metric CSV + key numbers
    out = [f"# ncu --set full captures, round {tag}", ""]
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem"]
    for f in sorted(os.listdir(GO)):
        if not (f.startswith(f"prof_{tag}_") and f.endswith(".ncu-rep")) or (
                sys.argv[2:] and not any(k in f for k in sys.argv[2:])):
            continue
        raw = subprocess.run(["ncu", "-i", os.path.join(GO, f), "--page", "raw", "--csv"],
                             capture_output=True, text=True).stdout
        stem = f[:-len(".ncu-rep")]
        open(os.path.join(PR, stem + "_raw.csv"), "w").write(raw)
        rows = list(csv.reader(raw.splitlines()))
        hdr, units, vals = rows[0], rows[1], rows[2]
        out += [f"## {stem}", "", "| metric | value |", "|---|---:|"]
        for h, u, v in zip(hdr, units, vals):
            if h in keys or (h.startswith("smsp__pcsamp_warps_issue_stalled") and
                             not h.endswith("not_issued") and v not in ("0", "")):
                out.append(f"| {h} ({u}) | {v} |")
        out.append("")
    open(os.path.join(PR, f"ncu_{tag}_summary.md"), "w").write("\n".join(out) + "\n")
    print("wrote", PR)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
