#!/usr/bin/env python3
"""Fixed vs per-pixel cost of each program: steady-state launch time (median of
ROUNDS groups of G back-to-back launches) over several square sizes, and the
least-squares fit t = a + b * N^2 (a = fixed cost per launch: ramp-up, tail,
launch gap; 8 / b = marginal HBM bandwidth).
usage: python tools/size_sweep.py 4096,8192,12288,16384 wavelet/scheme[/fwd|inv] ..."""
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1605_00561_b200 as wl  # noqa: E402

sizes = [int(x) for x in sys.argv[1].split(",")]
if os.environ.get("ENGINE"):  # 1 = generic interpreter, 3 = fast engine direct-load variant
    wl.set_engine(int(os.environ["ENGINE"]))
G = int(os.environ.get("G", "10"))
ROUNDS = int(os.environ.get("ROUNDS", "7"))
SLEEP = int(os.environ.get("SLEEP", "4000000"))  # cycles (~2 ms) of GPU sleep before each group
bufs = {}
for n in sizes:
    img = torch.rand((n, n), device="cuda")
    bufs[n] = (img, torch.empty((4, n // 2, n // 2), device="cuda"), torch.empty_like(img))
for prog in sys.argv[2:]:
    parts = prog.split("/")
    w, s = parts[0], parts[1]
    sch = wl.build_scheme(s, w)
    for d in ([parts[2]] if len(parts) > 2 else ["fwd", "inv"]):
        pts = []
        for n in sizes:
            img, q, rec = bufs[n]
            wl.forward(img, sch, out=q)

            def call():
                if d == "fwd":
                    wl.forward(img, sch, out=q)
                else:
                    wl.inverse(q, w, scheme=s, out=rec)
            for _ in range(3):
                call()
            ts = []
            for _ in range(ROUNDS):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda._sleep(SLEEP)  # the group is enqueued while the GPU sleeps:
                e0.record()               # no host launch latency inside the timed region
                for _ in range(G):
                    call()
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1) / G)
            pts.append((n * n, statistics.median(ts)))
        xs, ys = [p[0] for p in pts], [p[1] for p in pts]
        mx, my = sum(xs) / len(xs), sum(ys) / len(ys)
        b = sum((x - mx) * (y - my) for x, y in zip(xs, ys)) / sum((x - mx) ** 2 for x in xs)
        a = my - b * mx
        line = " ".join(f"{int(x ** 0.5)}:{y:.4f}" for x, y in pts)
        print(f"{w}/{s}/{d:3s} {line} | fixed {a * 1e3:6.1f} us  marginal {8 / (b * 1e-3) / 1e9:7.1f} GB/s",
              flush=True)
