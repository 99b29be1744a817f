"""The product's scheme algebra (paper_1605_00561_b200/schemes.py, the source
of every kernel constant) against the reference's own build_scheme output
(tests/golden/schemes_ref.json, dumped from the unmodified reference)."""
import json
import os
import subprocess
import sys
from fractions import Fraction

import pytest

from paper_1605_00561_b200 import schemes as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = json.load(open(os.path.join(ROOT, "tests", "golden", "schemes_ref.json")))


def _norm(poly, exact):
    return sorted((t[0], t[1], Fraction(t[2]) if exact else t[3]) for t in poly)


@pytest.mark.parametrize("wavelet", S.WAVELETS)
@pytest.mark.parametrize("scheme", S.SCHEMES)
def test_scheme_matches_reference_dump(wavelet, scheme):
    mine = S.build_scheme(scheme, wavelet)
    r = REF[wavelet][scheme]
    exact = bool(r["exact"])
    assert mine.barriers == r["barriers"] and mine.macs == r["macs"]
    assert [s.label for s in mine.steps] == [s["label"] for s in r["steps"]]
    assert [int(s.barrier) for s in mine.steps] == [s["barrier"] for s in r["steps"]]
    assert [s.kind for s in mine.steps] == [s["kind"] for s in r["steps"]]
    for st, rs in zip(mine.steps, r["steps"]):
        want = {(e[0], e[1]): _norm(e[2], exact) for e in rs["entries"]}
        got = {k: sorted((km, kn, v if exact else float(v)) for (km, kn), v in p.items())
               for k, p in st.matrix.items() if p}
        assert got == want, (wavelet, scheme, st.label)
    if scheme == "convolution":
        assert [sorted((k[0], k[1], v if exact else float(v)) for k, v in f.items())
                for f in mine.conv] == [_norm(f, exact) for f in r["conv"]]


def _product(steps, one):
    acc = {(i, i): {(0, 0): one} for i in range(4)}
    for st in steps:
        acc = S.m_mul(st.matrix, acc)
    return acc


@pytest.mark.parametrize("wavelet", ["cdf53", "cdf97", "dd137"])
@pytest.mark.parametrize("scheme", S.SCHEMES[:9])
def test_inverse_list_is_exact_inverse(wavelet, scheme):
    s = S.build_scheme(scheme, wavelet)
    one = s.wavelet.one
    prod = _product(s.steps + S.inverse_steps(s), one)
    for (i, j), p in prod.items():
        for k, v in p.items():
            want = 1 if (i == j and k == (0, 0)) else 0
            if s.wavelet.exact:
                assert v == want, (i, j, k, v)
            else:
                assert abs(v - want) < 1e-12, (i, j, k, v)
    # same number of neighbour epochs (= block barriers) as the forward
    assert len(S.epochs(S.inverse_steps(s))[1]) == len(S.epochs(s.steps)[1])


def test_generated_tables_are_current():
    gen = os.path.join(ROOT, "paper_1605_00561_b200", "csrc", "gen")
    before = {f: open(os.path.join(gen, f)).read() for f in os.listdir(gen)}
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "gen_steps.py")], check=True,
                   capture_output=True)
    after = {f: open(os.path.join(gen, f)).read() for f in os.listdir(gen)}
    assert before == after


def test_oracle_inverse_tables_agree_with_product():
    """Two independent derivations of the per-scheme inverse lists."""
    from oracle.oracle import inverse_step_list
    for w in ("cdf53", "cdf97"):
        for sch in S.SCHEMES[:9]:
            mine = S.inverse_steps(S.build_scheme(sch, w))
            theirs = inverse_step_list(w, sch)
            assert len(mine) == len(theirs)
            for a, b in zip(mine, theirs):
                ka = {k: p for k, p in a.matrix.items() if p}
                kb = {k: p for k, p in b.items() if p}
                assert set(ka) == set(kb)
                for k in ka:
                    assert set(ka[k]) == set(kb[k])
                    for t in ka[k]:
                        assert abs(float(ka[k][t]) - float(kb[k][t])) < 1e-14
