"""Periodic vs symmetric boundary, device time per transform (median of reps)."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1605_00561_b200 as wl  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
img = torch.rand((n, n), device="cuda")
q = torch.empty((4, n // 2, n // 2), device="cuda")
rec = torch.empty_like(img)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
for w, s in (("cdf53", "monolithic"), ("cdf97", "monolithic_star"), ("cdf97", "sweldens")):
    sch = wl.build_scheme(s, w)
    for b in ("periodic", "symmetric"):
        tf, ti = [], []
        for _ in range(12):
            ev[0].record()
            wl.forward(img, sch, b, out=q)
            ev[1].record()
            wl.inverse(q, w, b, scheme=s, out=rec)
            ev[2].record()
            torch.cuda.synchronize()
            tf.append(ev[0].elapsed_time(ev[1]))
            ti.append(ev[1].elapsed_time(ev[2]))
        print(f"{w}/{s} {b:9s} fwd {statistics.median(tf[2:]):.4f} ms  inv {statistics.median(ti[2:]):.4f} ms")
