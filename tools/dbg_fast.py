"""Runs each (wavelet, scheme, direction) of the fast engine once, syncing
after each, to localise a failing kernel: python tools/dbg_fast.py [size]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1605_00561_b200 as wl  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
wl.set_engine(2)
img = torch.rand((n, n), device="cuda")
for w in ("cdf53", "cdf97"):
    for s in ("monolithic_star", "sweldens"):
        sch = wl.build_scheme(s, w)
        q = wl.forward(img, sch)
        torch.cuda.synchronize()
        print(w, s, "fwd ok", flush=True)
        r = wl.inverse(q, w, scheme=s)
        torch.cuda.synchronize()
        print(w, s, "inv ok", (r - img).abs().max().item(), flush=True)
