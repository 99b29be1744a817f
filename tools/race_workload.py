"""Small fast-engine workload for compute-sanitizer racecheck / synccheck:
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
torch.cuda.synchronize()
print("workload done")
