"""Virtual-rank strip pyramids over sizes / rank counts (debug aid)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1605_00561_b200 as wl  # noqa: E402

sch = wl.build_scheme("monolithic_star", "cdf97")
for n in [int(x) for x in sys.argv[1].split(",")]:
    for ranks in [int(x) for x in sys.argv[2].split(",")]:
        img = torch.rand((n, n), device="cuda")
        rs = [wl.StripPyramid(n, n, 5, sch, r, ranks) for r in range(ranks)]
        if ranks > 1:
            blobs = [r.export() for r in rs]
            for r in range(ranks):
                rs[r].connect(blobs[(r - 1) % ranks], blobs[(r + 1) % ranks])
        rows = n // ranks
        for r in range(ranks):
            rs[r].input.copy_(img[r * rows:(r + 1) * rows])
        outs = [torch.empty(r.slice_elems(), device="cuda") for r in rs]
        torch.cuda.synchronize()
        streams = [torch.cuda.Stream() for _ in range(ranks)]
        t0 = time.time()
        for r in range(ranks):
            rs[r].forward(outs[r], stream=streams[r])
        torch.cuda.synchronize()
        ok = True
        try:
            for r in rs:
                r.check()
        except RuntimeError as e:
            ok = False
        print(f"n={n} ranks={ranks}: {'ok' if ok else 'TIMEOUT'} {time.time() - t0:.2f}s", flush=True)
        for r in rs:
            r.close()
