"""Host-buffer entry points: GPix/s of forward_host + inverse_host (pinned
buffers) for one program, wall clock. usage: python tools/bench_host.py [n] [reps]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1605_00561_b200 as wl  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
sch = wl.build_scheme("monolithic_star", "cdf97")
h = torch.rand((n, n)).pin_memory()
q = torch.empty((4, n // 2, n // 2)).pin_memory()
r = torch.empty((n, n)).pin_memory()
wl.forward_host(h, sch, out=q)
wl.inverse_host(q, "cdf97", scheme="monolithic_star", out=r)
t0 = time.perf_counter()
for _ in range(reps):
    wl.forward_host(h, sch, out=q)
t1 = time.perf_counter()
for _ in range(reps):
    wl.inverse_host(q, "cdf97", scheme="monolithic_star", out=r)
t2 = time.perf_counter()
gb = 4 * n * n / 1e9
print(f"chunk_kb={os.environ.get('WL_HOST_CHUNK_KB', 'default')} fwd {1e3 * (t1 - t0) / reps:.2f} ms "
      f"({gb / ((t1 - t0) / reps):.1f} GB/s each way) inv {1e3 * (t2 - t1) / reps:.2f} ms")
