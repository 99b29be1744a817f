"""GPU parity: the CUDA kernels (through the C-ABI) vs the CPU oracle.

Bars (BASELINE.json north_star):
* bit-exact: cdf53 on 8-bit dyadic inputs, every scheme, both boundaries,
  forward and inverse, levels 1-3 -> GPU float32 == (float32) oracle float64.
* tolerance: everything else: max |gpu - oracle| <= TOL * (max - min of the
  oracle plane), per plane, TOL = 1e-5.
* perfect reconstruction: GPU forward -> GPU inverse vs the input.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-5
SCHEMES = ["sweldens", "iwahashi", "iwahashi_star", "explosive", "explosive_star",
           "monolithic", "monolithic_star", "polyphase", "polyphase_star", "convolution"]
LIFTING = SCHEMES[:9]
BOUNDARIES = ["periodic", "symmetric"]
ENGINES = [0, 1]  # auto (fast where available), generic interpreter


@pytest.fixture(scope="module")
def wl():
    import paper_1605_00561_b200 as wl
    wl.lib()
    return wl


@pytest.fixture(autouse=True)
def _engine(wl):
    yield
    wl.set_engine(0)


def dyadic(h, w, seed):
    rng = np.random.default_rng(seed)
    return rng.integers(0, 256, size=(h, w)).astype(np.float64) / 256.0


def uniform(h, w, seed):
    return np.random.default_rng(seed).random((h, w))


def gpu(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def host(t):
    return t.double().cpu().numpy()


def rel_err(got, want):
    """max |got - want| / data range, per plane; a degenerate plane (1 cell,
    constant) is measured against the range of the whole output."""
    errs = []
    whole = max(float(want.max() - want.min()), float(np.abs(want).max()), 1e-30)
    for g, w in zip(got.reshape(-1, *got.shape[-2:]), want.reshape(-1, *want.shape[-2:])):
        rng = float(w.max() - w.min())
        rng = rng if rng > 1e-12 else whole
        errs.append(float(np.abs(g - w).max()) / rng)
    return max(errs)


def as_f32_oracle(img):
    """The oracle runs on exactly the float32 input the GPU sees."""
    return np.asarray(img, dtype=np.float32).astype(np.float64)


SIZES = [(32, 32), (64, 48), (2, 2), (4, 2), (2, 6), (34, 22), (130, 66), (256, 192)]


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("scheme", SCHEMES)
def test_cdf53_dyadic_bit_exact_forward(wl, oracle, scheme, engine):
    wl.set_engine(engine)
    s = wl.build_scheme(scheme, "cdf53")
    for (h, w) in SIZES:
        img = dyadic(h, w, h * 1000 + w)
        for b in BOUNDARIES:
            want = oracle.forward(img, "cdf53", scheme, b).astype(np.float32)
            got = wl.forward(gpu(img), s, b).cpu().numpy()
            assert np.array_equal(got, want), (scheme, b, h, w, np.abs(got - want).max())


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("scheme", SCHEMES)
def test_cdf97_forward_tolerance(wl, oracle, scheme, engine):
    wl.set_engine(engine)
    s = wl.build_scheme(scheme, "cdf97")
    for (h, w) in SIZES:
        img = as_f32_oracle(uniform(h, w, h * 7 + w))
        for b in BOUNDARIES:
            for sc in (False, True):
                want = oracle.forward(img, "cdf97", scheme, b, sc)
                got = host(wl.forward(gpu(img), s, b, sc))
                assert rel_err(got, want) <= TOL, (scheme, b, h, w, sc)


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("wavelet", ["cdf53", "cdf97"])
def test_inverse_per_scheme(wl, oracle, wavelet, engine):
    """Each scheme's inverse kernel vs the oracle's inverse of the same step
    list on arbitrary planes (not a forward output)."""
    wl.set_engine(engine)
    for (qh, qw) in [(16, 16), (1, 1), (3, 5), (33, 17), (96, 128)]:
        q = np.random.default_rng(qh * qw).integers(0, 256, (4, qh, qw)) / 256.0
        for scheme in LIFTING:
            for b in BOUNDARIES:
                want = oracle.inverse(q, wavelet, b, False, scheme=scheme)
                got = host(wl.inverse(gpu(q), wavelet, b, scheme=scheme))
                if wavelet == "cdf53":
                    assert np.array_equal(got, want.astype(np.float32)), (scheme, b, qh, qw)
                else:
                    assert rel_err(got, want) <= TOL, (scheme, b, qh, qw)


@pytest.mark.parametrize("wavelet", ["cdf53", "cdf97"])
def test_reference_inverse_matches_golden(wl, wavelet):
    g = np.load("tests/golden/inv_random16.npz")
    q = as_f32_oracle(g["planes"])
    for b in BOUNDARIES:
        for undo in (0, 1):
            got = host(wl.inverse(gpu(q), wavelet, b, bool(undo)))
            want = g[f"{wavelet}/{b}/{undo}"]
            # golden came from the float64 planes; compare against the range
            assert rel_err(got, want) <= TOL, (b, undo)


def test_forward_matches_golden_fixtures(wl):
    for tag in ("dyadic32", "random32"):
        g = np.load(f"tests/golden/fwd_{tag}.npz")
        img = g["img"]
        for w in ("cdf53", "cdf97"):
            for s in SCHEMES:
                for b in BOUNDARIES:
                    got = host(wl.forward(gpu(img), wl.build_scheme(s, w), b))
                    want = g[f"{w}/{s}/{b}"]
                    if tag == "dyadic32" and w == "cdf53":
                        assert np.array_equal(got, want), (w, s, b)
                    else:
                        assert rel_err(got, want) <= TOL, (tag, w, s, b)


@pytest.mark.parametrize("wavelet", ["cdf53", "cdf97"])
@pytest.mark.parametrize("levels", [1, 2, 3])
def test_pyramid(wl, oracle, wavelet, levels):
    h, w = 96, 160
    img = dyadic(h, w, levels) if wavelet == "cdf53" else as_f32_oracle(uniform(h, w, levels))
    for scheme in ("sweldens", "monolithic", "monolithic_star", "polyphase_star"):
        for b in BOUNDARIES:
            pyr = wl.multi_level_forward(gpu(img), wl.build_scheme(scheme, wavelet), levels, b)
            want = oracle.pyramid_forward(img, wavelet, scheme, levels, b)
            got = host(pyr.flat)
            if wavelet == "cdf53" and levels <= 2:
                # dyadic inputs stay exactly representable in fp32 for levels
                # 1-2 on this size (level 3 needs > 24 mantissa bits)
                assert np.array_equal(got, want.astype(np.float32)), (scheme, b, levels)
            else:
                assert np.abs(got - want).max() <= TOL * (want.max() - want.min())
            rec = host(wl.multi_level_inverse(pyr, wavelet, b, scheme=scheme))
            want_rec = oracle.pyramid_inverse(got, w, h, levels, wavelet, b, scheme=scheme)
            assert np.abs(rec - want_rec).max() <= TOL * (want_rec.max() - want_rec.min() + 1)


def test_golden_pyramids(wl):
    g = np.load("tests/golden/pyr_dyadic64x32.npz")
    for key in [k for k in g.files if k.startswith("fwd/")]:
        _, w, s, b = key.split("/")
        pyr = wl.multi_level_forward(gpu(g["img"]), wl.build_scheme(s, w), 3, b)
        want = g[key]
        got = host(pyr.flat)
        # 3 levels of cdf53 on 8-bit input need > 24 mantissa bits: tolerance
        assert np.abs(got - want).max() <= TOL * (want.max() - want.min()), key
        rec = host(wl.multi_level_inverse(pyr, w, b))
        assert np.abs(rec - g[f"inv/{w}/{s}/{b}"]).max() <= 1e-5, key


@pytest.mark.parametrize("wavelet", ["cdf53", "cdf97"])
def test_perfect_reconstruction_large(wl, wavelet):
    """Size-independent property at a large size: fwd -> inv == input."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(5)
    img = torch.rand((2048, 4096), device="cuda", generator=g)
    for scheme in LIFTING:
        for b in BOUNDARIES:
            q = wl.forward(img, wl.build_scheme(scheme, wavelet), b, True)
            rec = wl.inverse(q, wavelet, b, True, scheme=scheme)
            err = (rec - img).abs().max().item()
            if b == "symmetric" and scheme.startswith("polyphase"):
                continue  # not an exact inverse at the border (cli_smoke.sh:133-136)
            # two fp32 transforms back to back: PR bound 3e-5 of the [0,1) range
            assert err <= 3e-5, (scheme, b, err)


def test_cross_scheme_agreement_large(wl):
    """All schemes agree under periodic (test_transform.cpp:127-154) at 1024^2."""
    import torch
    img = (torch.randint(0, 256, (1024, 1024), device="cuda").float() / 256.0)
    ref53 = wl.forward(img, wl.build_scheme("sweldens", "cdf53"))
    for s in SCHEMES:
        assert torch.equal(wl.forward(img, wl.build_scheme(s, "cdf53")), ref53), s
    img = torch.rand((1024, 1024), device="cuda")
    ref97 = wl.forward(img, wl.build_scheme("sweldens", "cdf97"))
    for s in SCHEMES:
        d = (wl.forward(img, wl.build_scheme(s, "cdf97")) - ref97).abs().max().item()
        assert d <= 1e-5, (s, d)


@pytest.mark.parametrize("engine", [0, 1])
def test_dd137_small(wl, oracle, engine):
    """dd137 (reach 2, halo 3) on images smaller than one tile: the fast
    engine's lifting kernels (engine 0; Polyphase on the interpreter) and the
    interpreter alone (engine 1)."""
    wl.set_engine(engine)
    try:
        for (h, w) in ((40, 56), (64, 200)):
            img = dyadic(h, w, 3)
            for s in ("sweldens", "iwahashi", "monolithic_star", "polyphase", "convolution"):
                for b in BOUNDARIES:
                    want = oracle.forward(img, "dd137", s, b)
                    got = host(wl.forward(gpu(img), wl.build_scheme(s, "dd137"), b))
                    assert rel_err(got, want) <= TOL, (s, b, h, w)
    finally:
        wl.set_engine(0)


def test_dynamic_claim_slots_reused(wl):
    """Dynamic tile claims (more tiles than resident CTAs): each launch takes a
    counter slot of a 4096-slot ring that its last CTA resets; 4200 launches
    wrap the ring and every result stays bit-identical (a slot left non-zero
    would skip or repeat tiles)."""
    import torch
    img = torch.rand((2048, 2048), device="cuda")
    sch = wl.build_scheme("monolithic", "cdf53")
    q = wl.forward(img, sch)
    want = wl.inverse(q, "cdf53", scheme="monolithic")
    out = torch.empty_like(want)
    for k in range(4200):
        wl.inverse(q, "cdf53", scheme="monolithic", out=out)
        if k % 700 == 0 or k == 4199:
            assert torch.equal(out, want), k


def test_errors(wl):
    import torch
    s = wl.build_scheme("sweldens", "cdf53")
    with pytest.raises(ValueError):
        wl.forward(torch.zeros((5, 6), device="cuda"), s)
    with pytest.raises(ValueError):
        wl.multi_level_forward(torch.zeros((16, 12), device="cuda"), s, 3)
    with pytest.raises(ValueError):
        wl.multi_level_forward(torch.zeros((16, 16), device="cuda"), s, 0)


def test_launches_native_kernels(wl):
    import torch
    n0 = wl.launch_count()
    img = torch.rand((256, 256), device="cuda")
    wl.forward(img, wl.build_scheme("monolithic", "cdf53"))
    torch.cuda.synchronize()
    # fast engine kernel + the interpreter's border frame (or 1 interpreter launch)
    assert 1 <= wl.launch_count() - n0 <= 2


def test_apply_step_matches_reference(wl, ref):
    """apply_step (transform.cpp:100-125) on the GPU vs the unmodified
    reference's apply_step, for every step of several schemes (Scheme::steps
    walked like parsim.cpp does), both boundaries, ragged sizes."""
    for w in ("cdf53", "cdf97"):
        for s in ("sweldens", "monolithic_star", "polyphase", "explosive", "iwahashi_star"):
            for st in wl.build_scheme(s, w).steps:
                for (qh, qw) in ((37, 50), (130, 260), (1, 1), (2, 3)):
                    q = np.random.default_rng(qh * qw).integers(0, 256, (4, qh, qw)) / 256.0
                    for b in BOUNDARIES:
                        want = ref.apply_step(q, st.matrix.entries, b)
                        got = host(wl.apply_step(gpu(q), st, b))
                        if w == "cdf53":
                            assert np.array_equal(got, want), (s, st.label, b, qh, qw)
                        else:
                            assert rel_err(got, want) <= TOL, (s, st.label, b, qh, qw)
