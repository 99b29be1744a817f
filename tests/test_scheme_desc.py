"""The drop-in's Scheme::steps / conv_filters / scheme_step_matrices
(schemes.hpp:34-45,81) against the UNMODIFIED reference's build_scheme dump
(tests/golden/schemes_ref.json, made from oracle/_ref by tools/make_golden.py).
CPU only: host-side table queries through the C-ABI library."""
import pytest

import paper_1605_00561_b200 as wl
from oracle.oracle import _mmul, scheme_tables

WAVELETS = ["cdf53", "cdf97", "dd137"]
SCHEMES = ["sweldens", "iwahashi", "iwahashi_star", "explosive", "explosive_star",
           "monolithic", "monolithic_star", "polyphase", "polyphase_star", "convolution"]


@pytest.mark.parametrize("w", WAVELETS)
def test_steps_match_reference_build_scheme(w):
    for s in SCHEMES:
        ref = scheme_tables()[w][s]
        got = wl.build_scheme(s, w).steps
        assert len(got) == len(ref["steps"]), (w, s)
        for st, rs in zip(got, ref["steps"]):
            assert st.label == rs["label"], (w, s)
            assert st.matrix.kind == rs["kind"], (w, s, st.label)
            assert st.needs_barrier == bool(rs["barrier"]), (w, s, st.label)
            want = {}
            for row, col, terms in rs["entries"]:
                want[(row, col)] = [(km, kn, d) for km, kn, _, d in terms]
            have = {k: [(km, kn, c) for (km, kn), c in sorted(p.items())]
                    for k, p in st.matrix.entries.items()}
            assert have == want, (w, s, st.label)


@pytest.mark.parametrize("w", WAVELETS)
def test_conv_filters_match_reference(w):
    ref = scheme_tables()[w]["convolution"]["conv"]
    got = wl.build_scheme("convolution", w).conv_filters
    assert len(got) == 4
    for f, rf in zip(got, ref):
        assert sorted((km, kn, c) for (km, kn), c in f.items()) == \
            sorted((km, kn, d) for km, kn, _, d in rf)
    # tap counts (test_wavelets.cpp:177-185)
    if w == "cdf53":
        assert [len(f) for f in got] == [25, 15, 15, 9]
    if w == "cdf97":
        assert [len(f) for f in got] == [81, 63, 63, 49]
    assert wl.build_scheme("sweldens", w).conv_filters is None


@pytest.mark.parametrize("w", ["cdf53", "cdf97"])
def test_scheme_step_matrices(w):
    """schemes.cpp:221-228: Convolution's single matrix (the polyphase
    reassembly of its filters, polyphase.cpp:301-340) equals the product of
    the Sweldens steps -- the identity acceptance.cpp checks for every kind."""
    sw = wl.scheme_step_matrices(wl.build_scheme("sweldens", w))
    acc = sw[0].entries
    for m in sw[1:]:
        acc = _mmul(m.entries, acc)
    conv = wl.scheme_step_matrices(wl.build_scheme("convolution", w))
    assert len(conv) == 1
    got = conv[0].entries
    keys = set(acc) | set(got)
    for k in keys:
        a, b = acc.get(k, {}), got.get(k, {})
        for e in set(a) | set(b):
            assert abs(a.get(e, 0.0) - b.get(e, 0.0)) <= 1e-12, (w, k, e)


def test_errors():
    lib = wl.lib()
    assert lib.wl_scheme_nsteps(7, 0) == -1
    assert lib.wl_scheme_step(0, 0, 99, None, None, None, None, 0) == wl.WL_EINVAL
    assert lib.wl_scheme_conv_filter(0, 4, None, None, None, 0) == -1
    assert lib.wl_scheme_nsteps(0, 9) == 0  # Convolution has no steps
