"""bench.py's configs[1] step alone (40 programs, 8192^2), device time per
step: python tools/bench_step.py [steps]  (WL_LIB picks a variant)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1605_00561_b200 as wl  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
n = 8192
img = torch.rand((n, n), device="cuda")
q = torch.empty((4, n // 2, n // 2), device="cuda")
rec = torch.empty_like(img)
progs = [(w, s) for w in ("cdf53", "cdf97") for s in wl.SCHEMES]
sch = {p: wl.build_scheme(p[1], p[0]) for p in progs}


def step():
    for (w, s) in progs:
        wl.forward(img, sch[(w, s)], out=q)
        wl.inverse(q, w, scheme=s, out=rec)


for _ in range(3):
    step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(steps):
    step()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
print(f"{os.environ.get('WL_LIB', 'base')}: step {ms:.3f} ms  {80 * n * n / 2 / ms / 1e6:.1f} GPix/s")
