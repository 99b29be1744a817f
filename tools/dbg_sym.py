"""Symmetric-boundary fast path vs the CPU oracle: max error and where."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1605_00561_b200 as wl  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402

orc = Oracle()
for (h, w) in [(32, 32), (64, 48), (96, 64), (130, 66), (256, 192), (512, 512)]:
    img = np.random.default_rng(h * 7 + w).random((h, w)).astype(np.float32).astype(np.float64)
    for wv in ("cdf53", "cdf97"):
        for s in ("sweldens", "monolithic_star", "polyphase"):
            for d in ("fwd", "inv"):
                if d == "fwd":
                    want = orc.forward(img, wv, s, "symmetric")
                    got = wl.forward(torch.from_numpy(img.astype(np.float32)).cuda(),
                                     wl.build_scheme(s, wv), "symmetric").double().cpu().numpy()
                else:
                    q = np.random.default_rng(h + w).random((4, h // 2, w // 2))
                    want = orc.inverse(q, wv, "symmetric", False, scheme=s)
                    got = wl.inverse(torch.from_numpy(q.astype(np.float32)).cuda(), wv,
                                     "symmetric", scheme=s).double().cpu().numpy()
                err = np.abs(got - want)
                i = np.unravel_index(err.argmax(), err.shape)
                bad = err.max() > 1e-4
                print(f"{h}x{w} {wv} {s} {d}: max err {err.max():.2e} at {i} {'BAD' if bad else ''}"
                      f" shape {want.shape}", flush=True)
