"""Small fast-engine workload (incl. the fused two-level launch) for
compute-sanitizer racecheck / synccheck:
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
# fused two-level pyramid launch (shared-memory task / completion hand-off)
if hasattr(wl.lib(), "wl_set_level_fusion"):
    wl.set_level_fusion(True)
    imgs = torch.rand((2, 128, 256), device="cuda")
    for w, s in (("cdf53", "sweldens"), ("cdf97", "monolithic_star")):
        wl.multi_level_forward_batch(imgs, wl.build_scheme(s, w), 2)
    wl.set_level_fusion(False)
torch.cuda.synchronize()
print("workload done")
