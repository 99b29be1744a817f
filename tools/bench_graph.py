"""configs[1] step: eager launches vs one CUDA graph replay (device time)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1605_00561_b200 as wl  # noqa: E402

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
s = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for mode in ("eager", "graph", "eager", "graph"):
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        g.replay() if mode == "graph" else step()
    e1.record()
    torch.cuda.synchronize()
    print(mode, f"{e0.elapsed_time(e1) / 10:.3f} ms/step")
rec2 = rec.clone()
step()
torch.cuda.synchronize()
print("graph == eager:", torch.equal(rec2, rec))
