"""Steady-state A/B timing of library variants in ONE process (same box, same
buffers, interleaved): each sample = one group of G back-to-back launches of a
program between two CUDA events (device time / G); median over rounds.
usage: python tools/ab_steady.py SIZE lib[,lib...] wavelet/scheme[/fwd|inv] ...
  (lib "base" = paper_1605_00561_b200/libwavelift_b200.so, "x" = ..._x.so)
env: G (launches per group, 10), ROUNDS (7)."""
import ctypes
import os
import statistics
import sys

# several builds of the same kernels in one process: load every module eagerly
# (with lazy loading a launch of one build's kernel can resolve to another's,
# whose large-shared-memory attribute was never set -> "invalid argument")
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import torch  # noqa: E402

SCHEMES = ["sweldens", "iwahashi", "iwahashi_star", "explosive", "explosive_star",
           "monolithic", "monolithic_star", "polyphase", "polyphase_star", "convolution"]
PKG = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_1605_00561_b200")
n = int(sys.argv[1])
tags = sys.argv[2].split(",")
G = int(os.environ.get("G", "10"))
ROUNDS = int(os.environ.get("ROUNDS", "7"))
SLEEP = int(os.environ.get("SLEEP", "4000000"))
P, I, L = ctypes.c_void_p, ctypes.c_int, ctypes.c_long
libs = []
for t in tags:
    path = os.path.join(PKG, "libwavelift_b200.so" if t == "base" else f"libwavelift_b200_{t}.so")
    lib = ctypes.CDLL(os.environ.get("WL_LIB_" + t, path))
    lib.wl_last_error.restype = ctypes.c_char_p
    lib.wl_dwt2_forward.argtypes = [P, I, I, L, I, I, I, I, P, P, P, P, L, P]
    lib.wl_dwt2_inverse.argtypes = [P, P, P, P, I, I, L, I, I, I, I, P, L, P]
    libs.append(lib)
img = torch.rand((n, n), device="cuda")
q = torch.empty((4, n // 2, n // 2), device="cuda")
rec = torch.empty_like(img)
peak = 6554.6
for prog in sys.argv[3:]:
    parts = prog.split("/")
    w, s = parts[0], parts[1]
    dirs = [parts[2]] if len(parts) > 2 else ["fwd", "inv"]
    wi, si = ["cdf53", "cdf97"].index(w), SCHEMES.index(s)
    for d in dirs:
        def call(lib):
            if d == "fwd":
                return lib.wl_dwt2_forward(img.data_ptr(), n, n, n, wi, si, 0, 0, q[0].data_ptr(),
                                           q[1].data_ptr(), q[2].data_ptr(), q[3].data_ptr(),
                                           n // 2, None)
            return lib.wl_dwt2_inverse(q[0].data_ptr(), q[1].data_ptr(), q[2].data_ptr(),
                                       q[3].data_ptr(), n // 2, n // 2, n // 2, wi, si, 0, 0,
                                       rec.data_ptr(), n, None)
        res = {t: [] for t in tags}
        for t, lib in zip(tags, libs):
            for _ in range(3):
                rc = call(lib)
                assert rc == 0, (t, prog, d, rc, lib.wl_last_error())
        for _ in range(ROUNDS):
            for t, lib in zip(tags, libs):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                call(lib)
                torch.cuda._sleep(SLEEP)  # enqueue the group while the GPU sleeps
                e0.record()
                for _ in range(G):
                    call(lib)
                e1.record()
                e1.synchronize()
                res[t].append(e0.elapsed_time(e1) / G)
        base = statistics.median(res[tags[0]])
        line = f"{n} {w}/{s}/{d:4s}"
        for t in tags:
            m = statistics.median(res[t])
            frac = 8.0 * n * n / (m * 1e-3) / 1e9 / peak
            line += f" | {t} {m:.4f} ms {frac:.3f}" + (f" x{m / base:.3f}" if t != tags[0] else "")
        print(line, flush=True)
