#!/usr/bin/env python3
"""Round-2 profile summaries (tools/profile_r02.sh outputs in gpurun_out/r02/)
into profiles/: traffic_r02.json (per-launch DRAM bytes for every program at
8192^2 and, keyed "c3/...", the configs[2] programs at 16384^2),
launches_r02.md, ncu_r02_summary.md and the raw metric pages of the full
captures."""
import collections
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from summarize_profiles import PROGRAMS, read_metrics_csv, short, to_bytes, to_us  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TAG = sys.argv[1] if len(sys.argv) > 1 else "r02"
GO = os.path.join(ROOT, "gpurun_out", TAG)
PR = os.path.join(ROOT, "profiles")
C3 = ["cdf97/monolithic_star", "cdf97/monolithic", "cdf97/sweldens", "cdf53/monolithic",
      "cdf53/monolithic_star"]


def traffic(path, progs, n, prefix=""):
    tr = read_metrics_csv(path)
    kern = [k for k in tr if "uniform_kernel" not in k[0] and "elementwise" not in k[0]]
    out = {}
    for i, p in enumerate(progs):
        pair = kern[8 * i + 6: 8 * i + 8]  # 3 warm-up pairs, then the timed pair
        for d, (name, m) in zip(("fwd", "inv"), pair):
            rb, wb = to_bytes(*m["dram__bytes_read.sum"]), to_bytes(*m["dram__bytes_write.sum"])
            out[f"{prefix}{p}/{d}"] = {"read": rb, "write": wb, "total": rb + wb,
                                       "algorithmic": 8.0 * n * n,
                                       "us": to_us(*m["gpu__time_duration.sum"]),
                                       "kernel": short(name)}
    return out


def main():
    t = traffic(os.path.join(GO, f"traffic_{TAG}.csv"), PROGRAMS, 8192)
    t.update(traffic(os.path.join(GO, f"traffic_c3_{TAG}.csv"), C3, 16384, "c3/"))
    json.dump({k: v["total"] for k, v in t.items()}, open(os.path.join(PR, f"traffic_{TAG}.json"), "w"),
              indent=1)
    ll = read_metrics_csv(os.path.join(GO, f"launches_{TAG}.csv"))
    agg = collections.defaultdict(list)
    for name, m in ll:
        if "spin_kernel" in name:  # torch.cuda._sleep before timed groups: not ours
            continue
        agg[short(name)].append(to_us(*m["gpu__time_duration.sum"]))
    tot = sum(sum(v) for v in agg.values())
    lines = [f"# ncu launch list, round {TAG}", "",
             "`ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv python "
             "bench.py --steps 1 --warmup 3 --no-c3 --no-c4 --no-c5 --e2e-steps 0 --no-cpu "
             f"--no-unaligned --no-dd137` (raw: `launches_{TAG}.csv`; tools/profile_r02.sh {TAG}). Cold-cache, "
             "serialised: compare shares, not absolutes.", "",
             "| kernel | launches | mean us | share of listed time |", "|---|---:|---:|---:|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| {k} | {len(v)} | {sum(v) / len(v):.1f} | {sum(v) / tot:.3f} |")
    lines += ["", f"## DRAM traffic per launch (`traffic_{TAG}.csv`, `traffic_c3_{TAG}.csv`)", "",
              "| program | kernel | read GB | write GB | total / algorithmic | us |",
              "|---|---|---:|---:|---:|---:|"]
    for p, v in t.items():
        lines.append(f"| {p} | {v['kernel']} | {v['read'] / 1e9:.3f} | {v['write'] / 1e9:.3f} | "
                     f"{v['total'] / v['algorithmic']:.3f} | {v['us']:.1f} |")
    open(os.path.join(PR, f"launches_{TAG}.md"), "w").write("\n".join(lines) + "\n")
    os.system(f"cp {os.path.join(GO, f'launches_{TAG}.csv')} {os.path.join(GO, f'traffic_{TAG}.csv')} "
              f"{os.path.join(GO, f'traffic_c3_{TAG}.csv')} {PR}/")
    # full captures: key metrics + stall breakdown + hot SASS
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem"]
    out = [f"# ncu --set full captures, round {TAG} (tools/profile_r02.sh {TAG})", ""]
    for f in sorted(os.listdir(GO)):
        if not (f.startswith(f"prof_{TAG}_") and f.endswith(".ncu-rep")):
            continue
        rep = os.path.join(GO, f)
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        stem = f[:-len(".ncu-rep")]
        open(os.path.join(PR, stem + "_raw.csv"), "w").write(raw)
        import csv
        rows = list(csv.reader(raw.splitlines()))
        hdr, units, vals = rows[0], rows[1], rows[2]
        out += [f"## {stem}", "", "| metric | value |", "|---|---:|"]
        for h, u, v in zip(hdr, units, vals):
            if h in keys or (h.startswith("smsp__pcsamp_warps_issue_stalled") and
                             not h.endswith("not_issued") and v not in ("0", "")):
                out.append(f"| {h} ({u}) | {v} |")
        src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                              "sass"], capture_output=True, text=True).stdout
        tmp = f"/tmp/{stem}_sass.csv"
        open(tmp, "w").write(src)
        hot = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sass_hot.py"), tmp, "12"],
                             capture_output=True, text=True).stdout
        out += ["", "```", hot.rstrip(), "```", ""]
    open(os.path.join(PR, f"ncu_{TAG}_summary.md"), "w").write("\n".join(out) + "\n")
    print("wrote", PR)


if __name__ == "__main__":
    main()
