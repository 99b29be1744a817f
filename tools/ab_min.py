"""Minimal A/B timing against any library build (only the core C-ABI entry
points, so older builds load too): median device time of forward / inverse.
usage: WL_LIB=path python tools/ab_min.py SIZE REPS wavelet/scheme ..."""
import ctypes
import os
import sys

import torch

SCHEMES = ["sweldens", "iwahashi", "iwahashi_star", "explosive", "explosive_star",
           "monolithic", "monolithic_star", "polyphase", "polyphase_star", "convolution"]
lib = ctypes.CDLL(os.environ["WL_LIB"])
n, reps = int(sys.argv[1]), int(sys.argv[2])
P, I, L = ctypes.c_void_p, ctypes.c_int, ctypes.c_long
lib.wl_dwt2_forward.argtypes = [P, I, I, L, I, I, I, I, P, P, P, P, L, P]
lib.wl_dwt2_inverse.argtypes = [P, P, P, P, I, I, L, I, I, I, I, P, L, P]
img = torch.rand((n, n), device="cuda")
q = torch.empty((4, n // 2, n // 2), device="cuda")
rec = torch.empty_like(img)
for prog in sys.argv[3:]:
    w, s = prog.split("/")
    wi, si = ["cdf53", "cdf97"].index(w), SCHEMES.index(s)
    fwd = lambda: lib.wl_dwt2_forward(img.data_ptr(), n, n, n, wi, si, 0, 0, q[0].data_ptr(),
                                      q[1].data_ptr(), q[2].data_ptr(), q[3].data_ptr(), n // 2,
                                      None)
    inv = lambda: lib.wl_dwt2_inverse(q[0].data_ptr(), q[1].data_ptr(), q[2].data_ptr(),
                                      q[3].data_ptr(), n // 2, n // 2, n // 2, wi, si, 0, 0,
                                      rec.data_ptr(), n, None)
    for name, fn in (("fwd", fwd), ("inv", inv)):
        for _ in range(3):
            assert fn() == 0
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        print(f"{os.path.basename(os.environ['WL_LIB']):28s} {prog}/{name:4s} {ts[len(ts) // 2]:.4f} ms",
              flush=True)
