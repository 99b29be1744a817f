"""Pyramid drivers: eager launches vs graph replay (wl_set_graphs), device
time per call of back-to-back calls and host time per call.
usage: python tools/bench_pyr_graph.py"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1605_00561_b200 as wl  # noqa: E402

for (n, levels, w) in ((1024, 5, "cdf53"), (2048, 5, "cdf97"), (4096, 3, "cdf97"),
                       (8192, 5, "cdf97")):
    img = torch.rand((n, n), device="cuda")
    sch = wl.build_scheme("monolithic_star", w)
    out = torch.empty(n * n, device="cuda")
    scr = torch.empty(wl.lib().wl_pyramid_scratch_elems(n, n, levels), device="cuda")
    rec = torch.empty_like(img)
    pyr = wl.Pyramid(out, n, n, levels)
    res = {}
    for mode in (False, True, False, True):
        wl.set_graphs(mode)
        for _ in range(3):
            wl.multi_level_forward(img, sch, levels, out=out, scratch=scr)
            wl.multi_level_inverse(pyr, w, scheme="monolithic_star", out=rec, scratch=scr)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 50
        t0 = time.perf_counter()
        e0.record()
        for _ in range(reps):
            wl.multi_level_forward(img, sch, levels, out=out, scratch=scr)
            wl.multi_level_inverse(pyr, w, scheme="monolithic_star", out=rec, scratch=scr)
        e1.record()
        host = (time.perf_counter() - t0) / reps * 1e3
        torch.cuda.synchronize()
        res[mode] = (e0.elapsed_time(e1) / reps, host)
    print(f"{n}^2 {levels} levels {w}: eager {res[False][0]:.4f} ms/pair (host {res[False][1]:.4f})"
          f" | graph {res[True][0]:.4f} ms/pair (host {res[True][1]:.4f})", flush=True)
