"""GPU: batched transforms (BASELINE configs[4]) and row-strip transforms
(configs[3]) against the single-image path and the CPU oracle.

* batch: one launch over n images == n single-image calls, bit for bit
  (every wavelet x scheme x boundary; forward, inverse, pyramids).
* strips: the rows of a strip computed from the strip plus its halo rows ==
  the same rows of the whole-image transform (periodic), bit for bit; and the
  stitched strips match the oracle within the usual tolerance.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SCHEMES = ["sweldens", "iwahashi", "iwahashi_star", "explosive", "explosive_star",
           "monolithic", "monolithic_star", "polyphase", "polyphase_star", "convolution"]
LIFTING = SCHEMES[:9]
TOL = 1e-5


@pytest.fixture(scope="module")
def wl():
    import paper_1605_00561_b200 as wl
    wl.lib()
    return wl


@pytest.fixture(autouse=True)
def _engine(wl):
    yield
    wl.set_engine(0)


def rand(shape, seed, dyadic=False):
    import torch
    g = torch.Generator(device="cuda").manual_seed(seed)
    if dyadic:
        return torch.randint(0, 256, shape, device="cuda", generator=g).float() / 256.0
    return torch.rand(shape, device="cuda", generator=g)


@pytest.mark.parametrize("engine", [0, 1])
@pytest.mark.parametrize("wavelet", ["cdf53", "cdf97"])
def test_forward_batch_equals_single(wl, wavelet, engine):
    import torch
    wl.set_engine(engine)
    for (h, w) in [(64, 96), (130, 66), (256, 128)]:
        imgs = rand((3, h, w), h + w)
        for s in SCHEMES:
            sch = wl.build_scheme(s, wavelet)
            for b in ("periodic", "symmetric"):
                got = wl.forward_batch(imgs, sch, b, True)
                for i in range(3):
                    assert torch.equal(got[i], wl.forward(imgs[i], sch, b, True)), (s, b, h, w)


@pytest.mark.parametrize("wavelet", ["cdf53", "cdf97"])
def test_inverse_batch_equals_single(wl, wavelet):
    import torch
    for (qh, qw) in [(32, 48), (65, 33), (128, 64)]:
        q = rand((4, 4, qh, qw), qh * qw)
        for s in SCHEMES:
            for b in ("periodic", "symmetric"):
                got = wl.inverse_batch(q, wavelet, b, True, scheme=s)
                for i in range(4):
                    want = wl.inverse(q[i], wavelet, b, True, scheme=s)
                    assert torch.equal(got[i], want), (s, b, qh, qw)


@pytest.mark.parametrize("wavelet", ["cdf53", "cdf97"])
@pytest.mark.parametrize("levels", [1, 3])
def test_pyramid_batch_equals_single(wl, oracle, wavelet, levels):
    import torch
    h, w = 96, 160
    imgs = rand((3, h, w), levels, dyadic=True)
    for s in ("sweldens", "monolithic", "monolithic_star", "polyphase_star", "convolution"):
        sch = wl.build_scheme(s, wavelet)
        for b in ("periodic", "symmetric"):
            pyrs = wl.multi_level_forward_batch(imgs, sch, levels, b)
            for i in range(3):
                single = wl.multi_level_forward(imgs[i], sch, levels, b)
                assert torch.equal(pyrs[i], single.flat), (s, b)
            rec = wl.multi_level_inverse_batch(pyrs, w, h, levels, wavelet, b, scheme=s)
            for i in range(3):
                single = wl.multi_level_inverse(wl.Pyramid(pyrs[i].clone(), w, h, levels),
                                                wavelet, b, scheme=s)
                assert torch.equal(rec[i], single), (s, b)
    # and one image against the CPU oracle
    img = imgs[1].double().cpu().numpy()
    want = oracle.pyramid_forward(img, wavelet, "monolithic_star", levels, "periodic")
    got = wl.multi_level_forward_batch(imgs, wl.build_scheme("monolithic_star", wavelet),
                                       levels)[1].double().cpu().numpy()
    assert np.abs(got - want).max() <= TOL * (want.max() - want.min())


def strip_buffer(img, r0, r1, halo):
    """Rows [r0 - halo, r1 + halo) of a periodic image."""
    import torch
    h = img.shape[0]
    idx = torch.arange(r0 - halo, r1 + halo, device=img.device) % h
    return img[idx].contiguous()


@pytest.mark.parametrize("wavelet", ["cdf53", "cdf97"])
def test_forward_strips_equal_whole_image(wl, wavelet):
    import torch
    h, w = 288, 192
    img = rand((h, w), 11)
    halo = wl.strip_halo_rows(wavelet)
    for s in SCHEMES:
        sch = wl.build_scheme(s, wavelet)
        for sc in (False, True):
            whole = wl.forward(img, sch, "periodic", sc)
            for cuts in ([0, 96, 192, 288], [0, 2, 130, 288], [0, 288]):
                for r0, r1 in zip(cuts[:-1], cuts[1:]):
                    for extra in (0, 4):
                        buf = strip_buffer(img, r0, r1, halo + extra)
                        got = wl.forward_strip(buf, halo + extra, sch, sc)
                        want = whole[:, r0 // 2:r1 // 2]
                        assert torch.equal(got, want), (s, sc, r0, r1, extra)


@pytest.mark.parametrize("wavelet", ["cdf53", "cdf97"])
def test_inverse_strips_equal_whole_image(wl, wavelet):
    import torch
    qh, qw = 144, 96
    q = rand((4, qh, qw), 12)
    halo = wl.strip_halo_rows(wavelet, direction=1)
    for s in SCHEMES:
        for sc in (False, True):
            whole = wl.inverse(q, wavelet, "periodic", sc, scheme=s)
            for cuts in ([0, 48, 96, 144], [0, 1, 77, 144]):
                for r0, r1 in zip(cuts[:-1], cuts[1:]):
                    idx = torch.arange(r0 - halo, r1 + halo, device="cuda") % qh
                    buf = q[:, idx].contiguous()
                    got = wl.inverse_strip(buf, halo, wavelet, sc, scheme=s)
                    assert torch.equal(got, whole[2 * r0:2 * r1]), (s, sc, r0, r1)


def test_strip_errors(wl):
    import torch
    sch = wl.build_scheme("monolithic_star", "cdf97")
    buf = torch.zeros((64 + 4, 64), device="cuda")
    with pytest.raises(ValueError):
        wl.forward_strip(buf, 2, sch)  # halo below wl_strip_halo_rows (6 for cdf97)
    with pytest.raises(ValueError):
        wl.forward_strip(torch.zeros((64 + 12, 64), device="cuda"), 6,
                         wl.build_scheme("sweldens", "dd137"))
    assert wl.strip_halo_rows("cdf53") == 4 and wl.strip_halo_rows("cdf97") == 6


# ------------------------------------------------ row-strip pyramid (configs[3])
def _virtual_ranks(wl, img, levels, sch, n, calls=2):
    """n ranks in ONE process on one GPU (own stream each), connected through
    raw device pointers: exercises the halo protocol (push, flags, epochs)."""
    import torch
    h, w = img.shape
    ranks = [wl.StripPyramid(w, h, levels, sch, r, n) for r in range(n)]
    if n > 1:
        blobs = [r.export() for r in ranks]
        for r in range(n):
            ranks[r].connect(blobs[(r - 1) % n], blobs[(r + 1) % n])
    rows = h // n
    for r in range(n):
        ranks[r].input.copy_(img[r * rows:(r + 1) * rows])
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(n)]
    outs = [torch.full((ranks[r].slice_elems(),), float("nan"), device="cuda")
            for r in range(n)]
    torch.cuda.synchronize()
    for _ in range(calls):
        for r in range(n):
            ranks[r].forward(outs[r], stream=streams[r])
    torch.cuda.synchronize()
    for r in ranks:
        r.check()
        r.close()
    return wl.stitch_strip_pyramid(outs, w, h, levels)


@pytest.mark.parametrize("wavelet", ["cdf53", "cdf97"])
def test_strip_pyramid_virtual_ranks(wl, wavelet):
    import torch
    h, w, levels = 768, 256, 4
    img = rand((h, w), 21)
    for s in ("monolithic_star", "sweldens", "polyphase", "convolution"):
        sch = wl.build_scheme(s, wavelet)
        want = wl.multi_level_forward(img, sch, levels).flat
        for n in (1, 2, 3, 4):
            got = _virtual_ranks(wl, img, levels, sch, n)
            assert torch.equal(got, want), (s, n)


def _virtual_ranks_fwd_inv(wl, img, levels, sch, n, boundary):
    """Forward then inverse strip pyramid over n virtual ranks: (stitched
    flat pyramid, stitched reconstructed image)."""
    import torch
    h, w = img.shape
    ranks = [wl.StripPyramid(w, h, levels, sch, r, n, boundary=boundary) for r in range(n)]
    if n > 1:
        blobs = [r.export() for r in ranks]
        for r in range(n):
            ranks[r].connect(blobs[(r - 1) % n], blobs[(r + 1) % n])
    rows = h // n
    for r in range(n):
        ranks[r].input.copy_(img[r * rows:(r + 1) * rows])
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(n)]
    outs = [torch.full((ranks[r].slice_elems(),), float("nan"), device="cuda") for r in range(n)]
    recs = [torch.full((rows, w), float("nan"), device="cuda") for _ in range(n)]
    torch.cuda.synchronize()
    for _ in range(2):  # twice: the second call reuses the epoch protocol
        for r in range(n):
            ranks[r].forward(outs[r], stream=streams[r])
        for r in range(n):
            ranks[r].inverse(outs[r], out=recs[r], stream=streams[r])
    torch.cuda.synchronize()
    for r in ranks:
        r.check()
        r.close()
    return wl.stitch_strip_pyramid(outs, w, h, levels), torch.cat(recs)


@pytest.mark.parametrize("wavelet", ["cdf53", "cdf97"])
def test_strip_pyramid_symmetric_and_inverse(wl, wavelet):
    """Row strips under both boundaries, forward and inverse, vs the
    whole-image multi_level_forward / multi_level_inverse
    (transform.cpp:198-256): bit-identical where the arithmetic is exact
    (cdf53 dyadic) or the plans coincide (periodic); cdf97 symmetric within
    tolerance (the strip and the whole image may pick different border
    plans: mirrored register tiles vs interpreter frame)."""
    import torch
    h, w, levels = 768, 256, 4
    img = rand((h, w), 23, dyadic=(wavelet == "cdf53"))
    for s in ("monolithic_star", "sweldens", "iwahashi"):
        sch = wl.build_scheme(s, wavelet)
        for b in ("periodic", "symmetric"):
            want = wl.multi_level_forward(img, sch, levels, b).flat
            want_rec = wl.multi_level_inverse(wl.Pyramid(want, w, h, levels), wavelet, b,
                                              scheme=s)
            exact = wavelet == "cdf53" or b == "periodic"
            for n in (1, 2, 3, 4):
                got, rec = _virtual_ranks_fwd_inv(wl, img, levels, sch, n, b)
                if exact:
                    assert torch.equal(got, want), (s, b, n)
                    assert torch.equal(rec, want_rec), (s, b, n)
                else:
                    rng = (want.max() - want.min()).item()
                    assert (got - want).abs().max().item() <= TOL * rng, (s, b, n)
                    assert (rec - want_rec).abs().max().item() <= 3e-5, (s, b, n)
                if b == "periodic" or s != "polyphase":
                    assert (rec - img).abs().max().item() <= 3e-5, (s, b, n)


def test_strip_pyramid_errors(wl):
    sch = wl.build_scheme("monolithic_star", "cdf97")
    with pytest.raises(ValueError):
        wl.StripPyramid(256, 100, 2, sch, 0, 3)  # rows do not split evenly
    with pytest.raises(ValueError):
        wl.StripPyramid(256, 64, 4, sch, 0, 2)  # deepest strip thinner than the halo
    with pytest.raises(ValueError):
        wl.StripPyramid(256, 256, 2, wl.build_scheme("sweldens", "dd137"), 0, 1)
    with pytest.raises(ValueError):  # width not divisible by 2^levels
        wl.StripPyramid(1100, 1024, 3, sch, 0, 2)
    with pytest.raises(ValueError):  # symmetric strips need a lifting scheme
        wl.StripPyramid(256, 256, 2, wl.build_scheme("convolution", "cdf97"), 0, 2,
                        boundary="symmetric")


@pytest.mark.parametrize("wavelet", ["cdf53", "cdf97"])
def test_strip_pyramid_unaligned_levels(wl, wavelet):
    """Level widths 1160, 580, 290 px (= 0, 4, 2 mod 8): the deeper levels run
    the direct-load strip kernels (no TMA, halo wait in the exchange kernel);
    still bit-identical to the whole-image pyramid."""
    import torch
    img = rand((512, 1160), 22)
    sch = wl.build_scheme("monolithic_star", wavelet)
    want = wl.multi_level_forward(img, sch, 3).flat
    for n in (1, 2, 4):
        assert torch.equal(_virtual_ranks(wl, img, 3, sch, n), want), n


def _ipc_worker(rank, n, port, out_path):
    import torch
    import torch.distributed as dist
    import paper_1605_00561_b200 as wl
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=n)
    torch.cuda.set_device(0)
    h, w, levels = 512, 384, 3
    g = torch.Generator(device="cuda").manual_seed(77)
    img = torch.rand((h, w), device="cuda", generator=g)
    sch = wl.build_scheme("monolithic_star", "cdf97")
    rows = h // n
    sp = wl.strip_pyramid_distributed(img[rank * rows:(rank + 1) * rows], w, h, levels, sch)
    out = None
    for _ in range(3):
        out = sp.forward(out)
    torch.cuda.synchronize()
    sp.check()
    parts = [torch.empty(sp.slice_elems()) for _ in range(n)]
    dist.all_gather(parts, out.cpu())
    if rank == 0:
        got = wl.stitch_strip_pyramid(parts, w, h, levels)
        want = wl.multi_level_forward(img, sch, levels).flat.cpu()
        with open(out_path, "w") as f:
            f.write("ok" if torch.equal(got, want) else
                    f"mismatch {float((got - want).abs().max())}")
    dist.barrier()
    sp.close()
    dist.destroy_process_group()


def test_strip_pyramid_two_processes_ipc(tmp_path):
    """Two ranks = two processes sharing the one GPU: the halo goes through
    CUDA IPC peer memory exactly as between GPUs."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = tmp_path / "ipc.txt"
    mp.start_processes(_ipc_worker, args=(2, port, str(out)), nprocs=2, join=True,
                       start_method="spawn")
    assert out.read_text() == "ok"


# ------------------------------------------------------- host-buffer entry points
@pytest.mark.parametrize("wavelet", ["cdf53", "cdf97"])
def test_host_buffer_transforms_equal_device_path(wl, wavelet):
    """forward_host / inverse_host (pipelined row chunks) == the device path,
    bit for bit, including sizes with several chunks and a ragged last one."""
    import torch
    # (4100, 4100): w = 4 mod 8 px with several chunks -- no strip kernel for
    # that width, so the whole-image path must run (no WL_EINVAL)
    for (h, w) in [(8192 + 2 * 212, 1024), (512, 512), (34, 22), (4100, 4100)]:
        img = rand((h, w), h)
        for s in ("monolithic_star", "sweldens", "convolution", "polyphase"):
            sch = wl.build_scheme(s, wavelet)
            for b in ("periodic", "symmetric"):
                want = wl.forward(img, sch, b, True).cpu()
                got = wl.forward_host(img.cpu().pin_memory(), sch, b, True)
                assert torch.equal(got, want), (s, b, h, w)
                rec_want = wl.inverse(want.cuda(), wavelet, b, True, scheme=s).cpu()
                rec = wl.inverse_host(got.pin_memory(), wavelet, b, True, scheme=s)
                assert torch.equal(rec, rec_want), (s, b, h, w)


def test_strip_pyramid_large_virtual_ranks(wl):
    """configs[3] shape at scale: 16384^2, cdf97 Monolithic*, 5 levels, 4 strips
    (virtual ranks) == the whole-image pyramid, bit for bit."""
    import torch
    h = w = 16384
    img = rand((h, w), 33)
    sch = wl.build_scheme("monolithic_star", "cdf97")
    want = wl.multi_level_forward(img, sch, 5).flat
    got = _virtual_ranks(wl, img, 5, sch, 4, calls=1)
    assert torch.equal(got, want)
    del want, got
    torch.cuda.empty_cache()


def test_batch_pyramid_large(wl):
    """configs[4] shape: 16 images of 4096^2, 3 levels, batched == single calls."""
    import torch
    imgs = rand((16, 4096, 4096), 34)
    for w in ("cdf53", "cdf97"):
        sch = wl.build_scheme("monolithic_star", w)
        pyrs = wl.multi_level_forward_batch(imgs, sch, 3)
        for i in (0, 7, 15):
            assert torch.equal(pyrs[i], wl.multi_level_forward(imgs[i], sch, 3).flat), (w, i)
        rec = wl.multi_level_inverse_batch(pyrs, 4096, 4096, 3, w, scheme="monolithic_star")
        assert (rec - imgs).abs().max().item() <= 3e-5


def test_batch_beyond_int32_elements(wl):
    """Maximum sizes: one batched launch over 132 x 4096^2 images (2.2e9
    elements > 2^31): 64-bit image offsets in the kernels and 3-D TMA maps.
    The last images equal their single-image pyramids bit for bit."""
    import torch
    n = 132
    imgs = torch.empty((n, 4096, 4096), device="cuda")
    imgs[:-2].fill_(0.25)
    imgs[-2:] = rand((2, 4096, 4096), 35)
    sch = wl.build_scheme("monolithic_star", "cdf97")
    pyrs = wl.multi_level_forward_batch(imgs, sch, 2)
    for i in (n - 2, n - 1):
        assert torch.equal(pyrs[i], wl.multi_level_forward(imgs[i], sch, 2).flat), i
    assert torch.all(pyrs[0, -1024 * 1024:] == pyrs[0, -1]).item()  # constant image: flat LL
    del imgs, pyrs
    torch.cuda.empty_cache()


def test_strip_pyramid_forced_overlap():
    """The halo wait inside the strip transform (tile rows that read halo
    rows last, producer spins on the neighbours' flags) is only enabled by
    default when no neighbour shares the GPU; force it here so the one-GPU
    box exercises it: the small strip tests again, with WL_STRIP_OVERLAP=2.
    (Not the 16384^2 one: four ranks' persistent grids on ONE GPU can hold
    every SM while waiting for a neighbour's exchange kernel that then never
    gets scheduled -- the reason the default keeps the wait in the exchange
    kernel when a neighbour shares the device; the 10 s timeout turns that
    into an error, not a hang.)"""
    import os
    import subprocess
    import sys
    env = dict(os.environ, WL_STRIP_OVERLAP="2")
    here = os.path.abspath(__file__)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                        "-p", "no:cacheprovider", here, "-k",
                        "(virtual_ranks and not large) or two_processes_ipc"],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert " passed" in r.stdout
