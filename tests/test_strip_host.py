"""CPU: host-side logic of the row-strip pyramid (configs[3]) -- slice
layout and stitching (the ring exchange itself needs GPUs: see
test_gpu_batch_strip.py), plus the rank/neighbour ring over gloo."""
import numpy as np
import pytest
import torch

import paper_1605_00561_b200 as wl


def test_slice_layout_and_stitch_roundtrip():
    w, h, levels, n = 32, 48, 2, 3
    # a fake whole pyramid with distinct values, cut into rank slices by rows
    flat = torch.arange(w * h, dtype=torch.float32)
    planes, off = [], 0
    for l in range(levels):
        qw, qh = w >> (l + 1), h >> (l + 1)
        for _ in range(3):
            planes.append(flat[off:off + qw * qh].view(qh, qw))
            off += qw * qh
    qw, qh = w >> levels, h >> levels
    planes.append(flat[off:off + qw * qh].view(qh, qw))
    slices = []
    for r in range(n):
        parts = []
        for p in planes:
            rr = p.shape[0] // n
            parts.append(p[r * rr:(r + 1) * rr].reshape(-1))
        slices.append(torch.cat(parts))
    assert all(s.numel() == w * h // n for s in slices)
    assert torch.equal(wl.stitch_strip_pyramid(slices, w, h, levels), flat)
    views, ll = wl.strip_slice_planes(slices[1], w, h // n, levels)
    assert views[0][0].shape == (h // n // 2, w // 2) and ll.shape == (h // n // 4, w // 4)


def _ring_worker(rank, n, port, q):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=n)
    blobs = [None] * n
    dist.all_gather_object(blobs, f"blob{rank}".encode())
    q.put((rank, blobs[(rank - 1) % n], blobs[(rank + 1) % n]))
    dist.destroy_process_group()


def test_ring_neighbours_gloo():
    """The blob exchange strip_pyramid_distributed performs (world_size 2)."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_ring_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(60)
    assert res == [(0, b"blob1", b"blob1"), (1, b"blob0", b"blob0")]


def test_strip_validation_without_gpu():
    lib = wl.lib()
    import ctypes
    out = ctypes.c_void_p()
    assert lib.wl_strips_create(256, 100, 0, 3, 2, 1, 6, 0, ctypes.byref(out)) == wl.WL_EINVAL
    assert lib.wl_strips_create(256, 64, 0, 2, 4, 1, 6, 0, ctypes.byref(out)) == wl.WL_EINVAL
    assert lib.wl_strips_create(256, 256, 0, 1, 2, 2, 0, 0, ctypes.byref(out)) == wl.WL_EINVAL
    assert lib.wl_strip_halo_rows(1, 6, 0) == 6 and lib.wl_strip_halo_rows(2, 0, 0) == -1
