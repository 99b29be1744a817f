"""GPU: CUDA-graph replay of repeated pyramid calls (wl_set_graphs) gives the
same results as eager launches, counts its kernels, and keys on every
argument (a different buffer or shape is a different graph)."""
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def wl():
    import paper_1605_00561_b200 as wl
    wl.lib()
    return wl


@pytest.mark.parametrize("wavelet", ["cdf53", "cdf97"])
def test_graph_replay_equals_eager(wl, wavelet):
    import torch
    g = torch.Generator(device="cuda").manual_seed(3)
    for (h, w, levels) in ((512, 768, 3), (1024, 1024, 5), (96, 160, 2)):
        img = torch.rand((h, w), device="cuda", generator=g)
        for s in ("monolithic_star", "sweldens", "convolution"):
            sch = wl.build_scheme(s, wavelet)
            for b in ("periodic", "symmetric"):
                prev = wl.set_graphs(False)
                want = wl.multi_level_forward(img, sch, levels, b).flat.clone()
                wl.set_graphs(True)
                pyr = wl.Pyramid(torch.empty_like(want), w, h, levels)
                scratch = torch.empty(wl.lib().wl_pyramid_scratch_elems(w, h, levels),
                                      device="cuda")
                counts = []
                for _ in range(4):  # eager, capture + replay, replay, replay
                    pyr.flat.fill_(float("nan"))
                    n0 = wl.launch_count()
                    wl.multi_level_forward(img, sch, levels, b, out=pyr.flat, scratch=scratch)
                    torch.cuda.synchronize()
                    counts.append(wl.launch_count() - n0)
                    assert torch.equal(pyr.flat, want), (s, b, h, w)
                assert len(set(counts)) == 1 and counts[0] >= levels, counts
                wl.set_graphs(False)
                rec_want = wl.multi_level_inverse(pyr, wavelet, b, scheme=s)
                wl.set_graphs(True)
                rec = torch.empty_like(rec_want)
                for _ in range(3):
                    rec.zero_()
                    wl.multi_level_inverse(pyr, wavelet, b, scheme=s, out=rec, scratch=scratch)
                    assert torch.equal(rec, rec_want)
                wl.set_graphs(prev)


def test_graph_keys_on_arguments(wl):
    """Same shape, different output buffer -> the second buffer gets its own
    graph (and its own correct result)."""
    import torch
    sch = wl.build_scheme("monolithic", "cdf53")
    img = torch.rand((256, 256), device="cuda")
    outs = [torch.empty(256 * 256, device="cuda") for _ in range(2)]
    for _ in range(3):
        for o in outs:
            o.zero_()
            wl.multi_level_forward(img, sch, 3, out=o)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1]) and outs[0].abs().sum() > 0
