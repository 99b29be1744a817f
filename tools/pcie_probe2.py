"""PCIe duplex with the host pipeline's copy pattern: per chunk one 32 MB H2D
and four 8 MB D2H, 8 chunks, two streams (one per direction)."""
import time

import torch

MB = 1024 * 1024 // 4
h_in = torch.empty(256 * MB).pin_memory()
h_out = torch.empty(256 * MB).pin_memory()
d_in = torch.empty(256 * MB, device="cuda")
d_out = torch.empty(256 * MB, device="cuda")
si, so = torch.cuda.Stream(), torch.cuda.Stream()


def run(chunk_mb, pieces):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for k in range(256 // chunk_mb):
        a, b = k * chunk_mb * MB, (k + 1) * chunk_mb * MB
        with torch.cuda.stream(si):
            d_in[a:b].copy_(h_in[a:b], non_blocking=True)
        with torch.cuda.stream(so):
            step = (b - a) // pieces
            for p in range(pieces):
                h_out[a + p * step:a + (p + 1) * step].copy_(d_out[a + p * step:a + (p + 1) * step],
                                                            non_blocking=True)
    torch.cuda.synchronize()
    return time.perf_counter() - t


for _ in range(2):
    run(32, 4)
for chunk, pieces in ((256, 1), (32, 1), (32, 4), (8, 4), (64, 4)):
    t = min(run(chunk, pieces) for _ in range(3))
    print(f"chunk {chunk} MB, D2H in {pieces} pieces: {1.024 * 256 / 1000 / t * 1000 / 1.024:.1f} GB/s "
          f"per direction")
