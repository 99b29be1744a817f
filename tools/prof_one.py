"""Runs one (wavelet, scheme, direction) program a few times for ncu capture.
usage: python tools/prof_one.py cdf97 monolithic_star fwd 8192 [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1605_00561_b200 as wl  # noqa: E402

w, s, d, n = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
img = torch.rand((n, n), device="cuda")
sch = wl.build_scheme(s, w)
q = wl.forward(img, sch)
out = torch.empty_like(img)
for _ in range(reps):
    if d == "fwd":
        wl.forward(img, sch, out=q)
    else:
        wl.inverse(q, w, scheme=s, out=out)
torch.cuda.synchronize()
