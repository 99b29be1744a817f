"""Device time of one 2-level batched forward pyramid (fused or per-level).
usage: python tools/time_fused.py cdf53 4096 32"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1605_00561_b200 as wl  # noqa: E402

w, n, nb = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
img = torch.rand((nb, n, n), device="cuda")
sch = wl.build_scheme("monolithic_star", w)
out = wl.multi_level_forward_batch(img, sch, 2)
scratch = torch.empty(wl.lib().wl_pyramid_batch_scratch_elems(n, n, 2, nb), device="cuda")
ts = []
for _ in range(15):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    wl.multi_level_forward_batch(img, sch, 2, out=out, scratch=scratch)
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
print(f"{os.environ.get('TAG', '')} {w} {nb}x{n}^2 L2: {ts[len(ts) // 2]:.3f} ms")
