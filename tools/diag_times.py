#!/usr/bin/env python3
"""Where a persistent fast-engine launch spends its fixed cost: per-CTA
timestamps from a -DWL_DIAG_TIMES build (WL_LIB=..._diag.so).
usage: WL_LIB=paper_1605_00561_b200/libwavelift_b200_diag.so \
       python tools/diag_times.py SIZE wavelet/scheme/fwd|inv ..."""
import ctypes
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1605_00561_b200 as wl  # noqa: E402

n = int(sys.argv[1])
lib = wl.lib()
buf = torch.zeros(4 * 4096, dtype=torch.int64, device="cuda")
img = torch.rand((n, n), device="cuda")
q = torch.empty((4, n // 2, n // 2), device="cuda")
rec = torch.empty_like(img)
for prog in sys.argv[2:]:
    w, s, d = prog.split("/")
    sch = wl.build_scheme(s, w)
    wl.forward(img, sch, out=q)

    def call():
        if d == "fwd":
            wl.forward(img, sch, out=q)
        else:
            wl.inverse(q, w, scheme=s, out=rec)
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    rows = []
    for rep in range(5):
        buf.zero_()
        lib.wl_diag_set(ctypes.c_void_p(buf.data_ptr()))
        torch.cuda._sleep(2_000_000)
        call()   # previous launch of the same program right before: steady state
        call()
        torch.cuda.synchronize()
        lib.wl_diag_set(None)
        v = buf.view(-1, 4).cpu()
        v = v[v[:, 3] > 0]
        t0 = int(v[:, 0].min())
        ent = (v[:, 0] - t0).double() / 1e3
        first = (v[:, 1] - t0).double() / 1e3
        end = (v[:, 2] - t0).double() / 1e3
        tiles = v[:, 3].double()
        per_tile = ((end - first) / (tiles - 1).clamp(min=1)).median().item()
        rows.append((float(end.max()), float(ent.max()), float(first.median()), float(first.max()),
                     float(end.median()), float(end.min()), per_tile, float(tiles.min()),
                     float(tiles.max()), len(v)))
    r = [statistics.median(x) for x in zip(*rows)]
    print(f"{prog:28s} total {r[0]:6.1f} us | last entry {r[1]:5.1f} | first tile ready med {r[2]:5.1f} "
          f"max {r[3]:5.1f} | exit min {r[5]:6.1f} med {r[4]:6.1f} max {r[0]:6.1f} | "
          f"per tile {r[6]:5.2f} us | tiles/CTA {r[7]:.0f}-{r[8]:.0f} | CTAs {r[9]:.0f}", flush=True)
