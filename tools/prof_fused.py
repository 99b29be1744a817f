"""One fused two-level forward pyramid launch (or per-level with FUSE=0) for ncu.
usage: python tools/prof_fused.py cdf53 4096 32 [fuse=1]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1605_00561_b200 as wl  # noqa: E402

w, n, nb = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
fuse = int(sys.argv[4]) if len(sys.argv) > 4 else 1
wl.set_level_fusion(bool(fuse))
img = torch.rand((nb, n, n), device="cuda")
sch = wl.build_scheme("monolithic_star", w)
out = wl.multi_level_forward_batch(img, sch, 2)
scratch = torch.empty(wl.lib().wl_pyramid_batch_scratch_elems(n, n, 2, nb), device="cuda")
for _ in range(3):
    wl.multi_level_forward_batch(img, sch, 2, out=out, scratch=scratch)
torch.cuda.synchronize()
