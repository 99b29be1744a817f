#!/usr/bin/env python3
"""Per-program kernel timing for tuning (median of N reps, CUDA events).

usage: python tools/bench_kernels.py [size] [reps] [wavelet/scheme ...]
Prints one JSON line per program: median/min ms, GPix/s, HBM GB/s (8 B/px)
and the fraction of the measured copy peak.
"""
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1605_00561_b200 as wl  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
progs = sys.argv[3:] or ["cdf97/monolithic_star", "cdf97/monolithic", "cdf53/monolithic",
                         "cdf53/monolithic_star", "cdf97/sweldens"]
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
img = torch.rand((n, n), device="cuda")
q = torch.empty((4, n // 2, n // 2), device="cuda")
rec = torch.empty_like(img)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
for p in progs:
    w, s = p.split("/")
    sch = wl.build_scheme(s, w)
    for _ in range(3):
        wl.forward(img, sch, out=q)
        wl.inverse(q, w, scheme=s, out=rec)
    tf, ti = [], []
    for _ in range(reps):
        ev[0].record()
        wl.forward(img, sch, out=q)
        ev[1].record()
        wl.inverse(q, w, scheme=s, out=rec)
        ev[2].record()
        torch.cuda.synchronize()
        tf.append(ev[0].elapsed_time(ev[1]))
        ti.append(ev[1].elapsed_time(ev[2]))
    for d, t in (("fwd", tf), ("inv", ti)):
        med = statistics.median(t)
        gbs = 8.0 * n * n / (med * 1e-3) / 1e9
        print(json.dumps({"program": f"{p}/{d}", "size": n, "median_ms": round(med, 4),
                          "min_ms": round(min(t), 4), "gpix_s": round(n * n / med / 1e6, 1),
                          "hbm_gbs": round(gbs, 1), "frac": round(gbs / peak, 4)}), flush=True)
