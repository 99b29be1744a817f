"""Pins the CPU oracle (oracle/wl_oracle.c) before any GPU result is trusted.

1. Against the golden fixtures dumped from the UNMODIFIED reference
   (tests/golden/*, tools/make_golden.py): bit-identical float64.
2. Against the reference library itself (oracle/_ref) on fresh seeded
   inputs, including the reference tests' own cases
   (test_transform.cpp, acceptance.cpp).
"""
import numpy as np
import pytest

from oracle.oracle import BOUNDARIES, SCHEMES, inverse_step_list, forward_step_list

GOLD = "tests/golden/"


def test_resolve_index_tables(oracle):
    # proj/tests/test_transform.cpp:28-51
    p, s = "periodic", "symmetric"
    cases = [(0, 4, p, 0), (3, 4, p, 3), (4, 4, p, 0), (-1, 4, p, 3), (-5, 4, p, 3),
             (9, 4, p, 1), (0, 4, s, 0), (-1, 4, s, 1), (-2, 4, s, 2), (4, 4, s, 2),
             (5, 4, s, 1), (6, 4, s, 0), (7, 4, s, 1), (-5, 4, s, 1), (-3, 1, s, 0),
             (2, 1, s, 0), (-3, 1, p, 0)]
    for i, n, b, want in cases:
        assert oracle.resolve_index(i, n, b) == want


@pytest.mark.parametrize("tag", ["dyadic32", "random32"])
def test_forward_matches_golden(oracle, tag):
    g = np.load(GOLD + f"fwd_{tag}.npz")
    for w in ("cdf53", "cdf97"):
        for s in SCHEMES:
            for b in BOUNDARIES:
                got = oracle.forward(g["img"], w, s, b)
                assert np.array_equal(got, g[f"{w}/{s}/{b}"]), (w, s, b)


def test_scaling_matches_golden(oracle):
    g = np.load(GOLD + "fwd_scaled16.npz")
    for w in ("cdf53", "cdf97"):
        for b in BOUNDARIES:
            got = oracle.forward(g["img"], w, "sweldens", b, scaling=True)
            assert np.array_equal(got, g[f"{w}/sweldens/{b}"])


def test_inverse_matches_golden(oracle):
    g = np.load(GOLD + "inv_random16.npz")
    for w in ("cdf53", "cdf97"):
        for b in BOUNDARIES:
            for undo in (0, 1):
                got = oracle.inverse(g["planes"], w, b, bool(undo))
                assert np.array_equal(got, g[f"{w}/{b}/{undo}"]), (w, b, undo)


def test_pyramid_matches_golden(oracle):
    g = np.load(GOLD + "pyr_dyadic64x32.npz")
    for key in [k for k in g.files if k.startswith("fwd/")]:
        _, w, s, b = key.split("/")
        flat = oracle.pyramid_forward(g["img"], w, s, 3, b)
        assert np.array_equal(flat, g[key]), key
        rec = oracle.pyramid_inverse(flat, 64, 32, 3, w, b)
        assert np.array_equal(rec, g[f"inv/{w}/{s}/{b}"]), key


def test_dyadic_pyramid_exact_roundtrip(oracle):
    # test_transform.cpp:290-291: exact 3-level cdf53 reconstruction.
    g = np.load(GOLD + "pyr_dyadic64x32.npz")
    flat = oracle.pyramid_forward(g["img"], "cdf53", "sweldens", 3, "periodic")
    assert np.array_equal(oracle.pyramid_inverse(flat, 64, 32, 3, "cdf53"), g["img"])


@pytest.mark.parametrize("w", ["cdf53", "cdf97", "dd137"])
def test_forward_matches_reference_library(oracle, ref, w):
    for (iw, ih, seed) in ((64, 64, 7001), (18, 10, 5), (2, 2, 9), (6, 4, 3)):
        img = ref.random_image(iw, ih, seed)
        for s in SCHEMES:
            for b in BOUNDARIES:
                for sc in (False, True):
                    assert np.array_equal(oracle.forward(img, w, s, b, sc),
                                          ref.forward(img, w, s, b, sc)), (w, s, b, sc, iw, ih)


def test_inverse_matches_reference_library(oracle, ref):
    for w in ("cdf53", "cdf97", "dd137"):
        for (qw, qh) in ((8, 8), (9, 5), (1, 3)):
            q = ref.random_image(qw, 4 * qh, 77).reshape(4, qh, qw)
            for b in BOUNDARIES:
                for undo in (False, True):
                    assert np.array_equal(oracle.inverse(q, w, b, undo),
                                          ref.inverse(q, w, b, undo)), (w, qw, qh, b)


def test_apply_step_matches_reference_library(oracle, ref):
    """The per-scheme inverse steps through BOTH apply_step implementations."""
    q = ref.random_image(12, 40, 3).reshape(4, 10, 12)
    for w in ("cdf53", "cdf97"):
        for s in SCHEMES[:9]:
            for st in inverse_step_list(w, s) + forward_step_list(w, s):
                for b in BOUNDARIES:
                    assert np.allclose(oracle.apply_step(q, st, b), ref.apply_step(q, st, b),
                                       rtol=0, atol=1e-13)


def test_invalid_dimensions(oracle, ref):
    with pytest.raises(ValueError):
        oracle.forward(np.zeros((5, 6)), "cdf53", "sweldens")
    with pytest.raises(ValueError):
        ref.forward(np.zeros((5, 6)), "cdf53", "sweldens")
    with pytest.raises(ValueError):
        ref.pyramid_forward(np.zeros((16, 12)), "cdf53", "sweldens", 3)


def test_reference_cost_table(ref):
    # acceptance.cpp:62-67 frozen table
    want = {"cdf53": [(4, 16), (3, 24), (3, 18), (3, 24), (3, 18), (2, 24), (2, 18), (1, 63),
                      (1, 23), (1, 64)],
            "cdf97": [(8, 32), (6, 48), (6, 36), (6, 48), (6, 36), (4, 48), (4, 36), (2, 126),
                      (2, 46), (1, 256)]}
    for w, rows in want.items():
        for s, cell in zip(SCHEMES, rows):
            assert ref.cost(w, s) == cell
            assert ref.verify_identity(w, s)[0]


def test_per_scheme_inverse_is_exact_inverse(oracle, ref):
    """Oracle per-scheme inverse lists reconstruct the input (periodic all
    kinds; symmetric all non-polyphase kinds, cf. cli_smoke.sh:133-136)."""
    img = ref.random_image(32, 24, 11)
    for w in ("cdf53", "cdf97"):
        for s in SCHEMES[:9]:
            for b in BOUNDARIES:
                rec = oracle.inverse(oracle.forward(img, w, s, b), w, b, scheme=s)
                err = np.abs(rec - img).max()
                if b == "symmetric" and s.startswith("polyphase"):
                    continue
                assert err < 1e-12, (w, s, b, err)
