"""Per-level device time of batched forwards (the c5 pyramid's levels, one
launch each): n images of s^2 for s = S, S/2, S/4. usage: python tools/time_levels.py 64 4096"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1605_00561_b200 as wl  # noqa: E402

nb, S = int(sys.argv[1]), int(sys.argv[2])
peak = 6554.6
for w in ("cdf53", "cdf97"):
    sch = wl.build_scheme("monolithic_star", w)
    for s in (S, S // 2, S // 4):
        img = torch.rand((nb, s, s), device="cuda")
        out = wl.forward_batch(img, sch)
        ts = []
        for _ in range(12):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            wl.forward_batch(img, sch, out=out)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        ms = ts[len(ts) // 2]
        gbs = 8.0 * nb * s * s / ms / 1e6
        print(f"{w} {nb}x{s}^2 fwd: {ms:.3f} ms  {gbs:.0f} GB/s  {gbs / peak:.3f}", flush=True)
        del img, out
