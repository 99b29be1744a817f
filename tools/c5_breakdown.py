#!/usr/bin/env python3
"""configs[4] cost breakdown: one batched launch of 64 images per level size
(4096^2, 2048^2, 1024^2) vs the 3-level batched pyramid call, device time
behind a GPU sleep (steady state, median of 5 groups of 5).
usage: python tools/c5_breakdown.py [wavelet] [scheme]"""
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1605_00561_b200 as wl  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "cdf97"
s = sys.argv[2] if len(sys.argv) > 2 else "monolithic_star"
sch = wl.build_scheme(s, w)
nb, n, levels = 64, 4096, 3
imgs = torch.rand((nb, n, n), device="cuda")
pyr = torch.empty((nb, n * n), device="cuda")
scratch = torch.empty(wl.lib().wl_pyramid_batch_scratch_elems(n, n, levels, nb), device="cuda")


def timed(fn, groups=5, per=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(groups):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(4_000_000)
        e0.record()
        for _ in range(per):
            fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) / per)
    return statistics.median(ts)


peak = 6491.8
tot = 0.0
for lvl in range(levels):
    m = n >> lvl
    x = imgs[:, :m, :m].contiguous() if lvl else imgs
    q = torch.empty((nb, 4, m // 2, m // 2), device="cuda")
    t = timed(lambda: wl.forward_batch(x, sch, out=q))
    tot += t
    gbs = 8.0 * nb * m * m / (t * 1e-3) / 1e9
    print(f"level {lvl}: {nb} x {m}^2 one batched launch {t:.4f} ms  {gbs:.0f} GB/s  {gbs / peak:.3f}")
    del q
t = timed(lambda: wl.multi_level_forward_batch(imgs, sch, levels, out=pyr, scratch=scratch))
algo = 8.0 * nb * n * n * sum(4.0 ** -l for l in range(levels))
print(f"sum of single levels {tot:.4f} ms | 3-level pyramid call {t:.4f} ms "
      f"({algo / (t * 1e-3) / 1e9 / peak:.3f} of peak)")
