"""Batched pyramid (configs[4] shape) for ncu launch lists / per-level timing.
usage: python tools/prof_batch.py cdf97 [n_images] [levels] [size]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1605_00561_b200 as wl  # noqa: E402

w = sys.argv[1]
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 64
levels = int(sys.argv[3]) if len(sys.argv) > 3 else 3
n = int(sys.argv[4]) if len(sys.argv) > 4 else 4096
sch = wl.build_scheme("monolithic_star", w)
imgs = torch.rand((nb, n, n), device="cuda")
out = wl.multi_level_forward_batch(imgs, sch, levels)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for _ in range(3):
    ev[0].record()
    wl.multi_level_forward_batch(imgs, sch, levels, out=out)
    ev[1].record()
    torch.cuda.synchronize()
    print(w, nb, levels, n, "ms", ev[0].elapsed_time(ev[1]))
# single levels at each size, batched
for l in range(levels):
    s = n >> l
    x = torch.rand((nb, s, s), device="cuda")
    q = wl.forward_batch(x, sch)
    ts = []
    for _ in range(5):
        ev[0].record()
        wl.forward_batch(x, sch, out=q)
        ev[1].record()
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]))
    t = sorted(ts)[2]
    print(f"level {l} size {s}: {t:.4f} ms  {8 * nb * s * s / t / 1e6:.1f} GB/s")
