"""Small fast-engine workload (incl. dynamic tile claims and the reach-2
dd137 kernels) for compute-sanitizer racecheck / synccheck:
python tools/race_workload.py  (WL_LIB selects the library variant)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1605_00561_b200 as wl  # noqa: E402

wl.set_engine(2)  # fast engine only: the kernels with the per-epoch barriers
img = torch.rand((96, 512), device="cuda")
for w, s in (("cdf53", "sweldens"), ("cdf97", "monolithic_star")):
    sch = wl.build_scheme(s, w)
    for b in ("periodic", "symmetric"):  # symmetric: interior + mirroring border kernels
        q = wl.forward(img, sch, b)
        wl.inverse(q, w, b, scheme=s)
# more tiles than resident CTAs: the dynamic tile claims (producer -> compute
# warps task hand-off through shared memory) of the cdf53 / cdf97 inverse kernels
big = torch.rand((512, 4096), device="cuda")
for w, s in (("cdf53", "monolithic"), ("cdf97", "sweldens")):
    sch = wl.build_scheme(s, w)
    q = wl.forward(big, sch)
    wl.inverse(q, w, scheme=s)
# reach-2 dd137 kernels (two ghost rows, two-row edge exchange)
for s in ("sweldens", "monolithic_star"):
    q = wl.forward(img, wl.build_scheme(s, "dd137"))
    wl.inverse(q, "dd137", scheme=s)
torch.cuda.synchronize()
print("workload done")
