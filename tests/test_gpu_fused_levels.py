"""GPU: fused forward pyramid levels (two levels per persistent launch, the
coarser level reading the finer LL while it is still in L2)
== one launch per level, bit for bit, and == the CPU oracle.

The fused launch orders its tasks by dependency (level-l tile row j, then the
level-(l+1) tile rows whose LL_l rows are complete) and synchronises through
per-row completion counters; a wrong dependency shows up as a mismatch, so the
large cases are repeated.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

LIFTING = ["sweldens", "iwahashi", "iwahashi_star", "explosive", "explosive_star",
           "monolithic", "monolithic_star", "polyphase", "polyphase_star"]
TOL = 1e-5


@pytest.fixture(scope="module")
def wl():
    import paper_1605_00561_b200 as wl
    wl.lib()
    return wl


@pytest.fixture(autouse=True)
def _fusion(wl):
    prev = wl.set_level_fusion(True)
    yield
    wl.set_level_fusion(prev)
    wl.set_engine(0)


def rand(shape, seed):
    import torch
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.rand(shape, device="cuda", generator=g)


def both(wl, fn):
    wl.set_level_fusion(False)
    want = fn()
    wl.set_level_fusion(True)
    got = fn()
    return got, want


@pytest.mark.parametrize("wavelet", ["cdf53", "cdf97"])
def test_fused_equals_per_level(wl, wavelet):
    import torch
    for (h, w) in [(64, 64), (96, 160), (256, 1024), (1024, 768)]:
        img = rand((h, w), h + w)
        for s in LIFTING:
            sch = wl.build_scheme(s, wavelet)
            for levels in (2, 3, 5):
                if h % (1 << levels) or w % (1 << levels):
                    continue
                for scaling in (False, True):
                    got, want = both(wl, lambda: wl.multi_level_forward(
                        img, sch, levels, "periodic", scaling).flat)
                    assert torch.equal(got, want), (s, h, w, levels, scaling)


@pytest.mark.parametrize("wavelet", ["cdf53", "cdf97"])
def test_fused_batch_equals_per_level(wl, wavelet):
    import torch
    imgs = rand((5, 384, 512), 3)
    for s in ("sweldens", "monolithic_star", "polyphase"):
        sch = wl.build_scheme(s, wavelet)
        got, want = both(wl, lambda: wl.multi_level_forward_batch(imgs, sch, 3).clone())
        assert torch.equal(got, want), s


def test_fused_launch_count_and_oracle(wl, oracle):
    """4 levels -> 2 launches; the fused pyramid matches the CPU oracle."""
    import torch
    img = rand((512, 256), 9)
    for wavelet in ("cdf53", "cdf97"):
        sch = wl.build_scheme("monolithic_star", wavelet)
        torch.cuda.synchronize()
        n0 = wl.launch_count()
        got = wl.multi_level_forward(img, sch, 4).flat
        torch.cuda.synchronize()
        assert wl.launch_count() - n0 == 2
        want = oracle.pyramid_forward(img.double().cpu().numpy(), wavelet, "monolithic_star", 4,
                                      "periodic")
        g = got.double().cpu().numpy()
        assert np.abs(g - want).max() <= TOL * (want.max() - want.min())


def test_fused_large_repeated(wl):
    """16384^2 and 8192^2 pyramids, repeated: any dependency race would show
    up as a difference to the per-level result."""
    import torch
    for n, levels, wavelet in [(16384, 5, "cdf97"), (8192, 3, "cdf53")]:
        img = rand((n, n), n)
        sch = wl.build_scheme("monolithic_star", wavelet)
        wl.set_level_fusion(False)
        want = wl.multi_level_forward(img, sch, levels).flat.clone()
        wl.set_level_fusion(True)
        for _ in range(4):
            got = wl.multi_level_forward(img, sch, levels).flat
            assert torch.equal(got, want), (n, wavelet)
        del img, want, got
        torch.cuda.empty_cache()
