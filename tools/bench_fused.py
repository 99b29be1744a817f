"""Fused vs per-level forward pyramids (device-resident, CUDA events, median).
usage: python tools/bench_fused.py [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1605_00561_b200 as wl  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10


def timeit(fn):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


cases = [("single", 16384, 1, 5), ("single", 8192, 1, 3), ("batch", 4096, 32, 3),
         ("single", 32768, 1, 5)]
for kind, n, nb, levels in cases:
    for wavelet in ("cdf53", "cdf97"):
        sch = wl.build_scheme("monolithic_star", wavelet)
        if kind == "single":
            img = torch.rand((n, n), device="cuda")
            out = wl.multi_level_forward(img, sch, levels).flat
            scratch = torch.empty(wl.lib().wl_pyramid_scratch_elems(n, n, levels), device="cuda")

            def fn():
                wl.lib().wl_dwt2_pyramid_forward(
                    img.data_ptr(), n, n, levels, sch.wavelet.index, sch.kind, 0, 0,
                    out.data_ptr(), scratch.data_ptr(), None)
        else:
            img = torch.rand((nb, n, n), device="cuda")
            out = wl.multi_level_forward_batch(img, sch, levels)
            scratch = torch.empty(wl.lib().wl_pyramid_batch_scratch_elems(n, n, levels, nb),
                                  device="cuda")

            def fn():
                wl.multi_level_forward_batch(img, sch, levels, out=out, scratch=scratch)
        res = []
        for fuse in (False, True):
            wl.set_level_fusion(fuse)
            res.append(timeit(fn))
        wl.set_level_fusion(True)
        byts = 8.0 * n * n * nb * sum(4.0 ** -l for l in range(levels))
        print(f"{kind:6s} {nb:3d}x{n:5d}^2 L{levels} {wavelet}: per-level {res[0]:8.3f} ms "
              f"({byts / res[0] / 1e6:6.0f} GB/s)  fused {res[1]:8.3f} ms "
              f"({byts / res[1] / 1e6:6.0f} GB/s)  x{res[0] / res[1]:.3f}", flush=True)
        del img, out, scratch
        torch.cuda.empty_cache()
