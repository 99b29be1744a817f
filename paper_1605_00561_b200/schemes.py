"""Scheme catalogue for the B200 kernels (host-side constant generation).

This is the product's own restatement of the reference's wavelet and scheme
algebra -- the *selection surface* of the drop-in API -- used at BUILD time to
generate the per-(wavelet, scheme, direction) constant tables and the
straight-line register code of the CUDA kernels
(``tools/gen_steps.py`` -> ``csrc/gen/*.h``). Nothing here runs per pixel.

Reference correspondences (``/root/reference/proj``):

* wavelets: ``src/wavelets.cpp:27-62`` (``get_wavelet``), ``:65-74``
  (``split_operators``), ``laurent.cpp:93-103`` (``split_scalar``)
* step matrices: ``src/polyphase.cpp:75-171`` (``build_matrix``, 13 kinds)
* schemes: ``src/schemes.cpp:17-37`` (names), ``:49-142`` (base/star stage
  lists), ``:146-174`` (``build_scheme``), ``:176-198`` (cost counts)
* tap convention: ``include/wavelift/laurent.hpp:5-15`` -- exponent (k_m, k_n)
  reads component sample (row - k_n, col - k_m).

The generated tables are checked entry-for-entry against the reference's own
``build_scheme`` output (``tests/golden/schemes_ref.json``, dumped from the
unmodified reference) in ``tests/test_schemes.py``.

Inverse step lists (a per-scheme inverse the reference does not have; its
``inverse`` is wavelet-only, ``transform.cpp:178-196``) are the forward list
reversed with every step inverted exactly: ``I - N + N^2 - ...`` for the
unipotent kinds and the negated reversed Sweldens product for ``N_FULL``.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from fractions import Fraction

WAVELETS = ("cdf53", "cdf97", "dd137")
SCHEMES = ("sweldens", "iwahashi", "iwahashi_star", "explosive", "explosive_star",
           "monolithic", "monolithic_star", "polyphase", "polyphase_star", "convolution")
BOUNDARIES = ("periodic", "symmetric")
LL, HL, LH, HH = 0, 1, 2, 3
COMP_NAMES = ("LL", "HL", "LH", "HH")


# ----------------------------------------------------------- Laurent algebra
# 1-D polynomial: {exponent: coeff}; 2-D: {(k_m, k_n): coeff}. Zero terms are
# never stored (laurent.hpp:11-13), so tap counts are well defined.

def _clean(p):
    return {k: v for k, v in p.items() if v != 0}


def p_add(a, b):
    r = dict(a)
    for k, v in b.items():
        r[k] = r.get(k, 0) + v
    return _clean(r)


def p_neg(a):
    return {k: -v for k, v in a.items()}


def p_mul1(a, b):
    r = {}
    for ka, va in a.items():
        for kb, vb in b.items():
            r[ka + kb] = r.get(ka + kb, 0) + va * vb
    return _clean(r)


def p_mul2(a, b):
    r = {}
    for (am, an), va in a.items():
        for (bm, bn), vb in b.items():
            k = (am + bm, an + bn)
            r[k] = r.get(k, 0) + va * vb
    return _clean(r)


def orient_h(p):
    """laurent.cpp:216-225 orient(p, horizontal): k -> (k, 0)."""
    return {(k, 0): v for k, v in p.items()}


def transpose(p):
    """laurent.cpp:184-188: (k_m, k_n) -> (k_n, k_m)."""
    return {(kn, km): v for (km, kn), v in p.items()}


def is_one(p):
    return len(p) == 1 and p.get((0, 0), 0) == 1


def split_scalar(p):
    """laurent.cpp:93-103: (exponent-0 part, residual)."""
    return ({k: v for k, v in p.items() if k == 0}, {k: v for k, v in p.items() if k != 0})


# ------------------------------------------------------------------ wavelets
@dataclass
class Wavelet:
    name: str
    stages: list          # [(predict, update)] 1-D polys
    zeta: float
    exact: bool

    @property
    def one(self):
        return Fraction(1) if self.exact else 1.0


def get_wavelet(name: str) -> Wavelet:
    """wavelets.cpp:27-62."""
    F = Fraction
    if name == "cdf53":
        return Wavelet(name, [({0: F(-1, 2), -1: F(-1, 2)}, {0: F(1, 4), 1: F(1, 4)})],
                       math.sqrt(2.0), True)
    if name == "cdf97":
        alpha, beta = -1.5861343420693648, -0.052980118572961
        gamma, delta = 0.882911075530934, 0.443506852043971
        return Wavelet(name, [({0: alpha, -1: alpha}, {0: beta, 1: beta}),
                              ({0: gamma, -1: gamma}, {0: delta, 1: delta})],
                       1.149604398860241, False)
    if name == "dd137":
        return Wavelet(name, [({1: F(1, 16), -2: F(1, 16), 0: F(-9, 16), -1: F(-9, 16)},
                               {0: F(9, 32), 1: F(9, 32), -1: F(-1, 32), 2: F(-1, 32)})],
                       1.0, True)
    raise ValueError(f"unknown wavelet: {name}")


# ------------------------------------------------------------- step matrices
MATRIX_KINDS = ("T_H", "T_V", "S_H", "S_V", "T_I", "R_I", "S_I", "T_E", "R_E", "S_E",
                "T_MONO", "S_MONO", "N_FULL")


def build_matrix(kind: str, predict: dict, update: dict, one) -> dict:
    """polyphase.cpp:75-171. Returns {(dst, src): 2-D poly} incl. the identity
    diagonal. `predict`/`update` are 1-D polys (empty = zero operator)."""
    ph = orient_h(predict)
    pv = transpose(ph)
    uh = orient_h(update)
    uv = transpose(uh)
    m = {(i, i): {(0, 0): one} for i in range(4)}

    def put(r, c, p):
        if p:
            m[(r, c)] = p
        else:
            m.pop((r, c), None)

    if kind == "T_H":
        put(HL, LL, ph); put(HH, LH, ph)
    elif kind == "T_V":
        put(LH, LL, pv); put(HH, HL, pv)
    elif kind == "S_H":
        put(LL, HL, uh); put(LH, HH, uh)
    elif kind == "S_V":
        put(LL, LH, uv); put(HL, HH, uv)
    elif kind == "T_I":
        put(HH, LL, p_mul2(ph, pv)); put(HH, HL, pv); put(HH, LH, ph)
    elif kind == "R_I":
        put(HL, LL, ph); put(HL, HH, uv); put(LH, LL, pv); put(LH, HH, uh)
    elif kind == "S_I":
        put(LL, HL, uh); put(LL, LH, uv); put(LL, HH, p_neg(p_mul2(uh, uv)))
    elif kind == "T_E":
        put(HL, LL, ph); put(LH, LL, pv); put(HH, LL, p_neg(p_mul2(ph, pv)))
    elif kind == "R_E":
        put(LL, HL, uh); put(LL, LH, uv); put(HH, HL, pv); put(HH, LH, ph)
    elif kind == "S_E":
        put(LL, HH, p_mul2(uh, uv)); put(HL, HH, uv); put(LH, HH, uh)
    elif kind == "T_MONO":
        put(HL, LL, ph); put(LH, LL, pv); put(HH, LL, p_mul2(ph, pv))
        put(HH, HL, pv); put(HH, LH, ph)
    elif kind == "S_MONO":
        put(LL, HL, uh); put(LL, LH, uv); put(LL, HH, p_mul2(uh, uv))
        put(HL, HH, uv); put(LH, HH, uh)
    elif kind == "N_FULL":
        v1 = p_add(p_mul1(predict, update), {0: one})
        vh = orient_h(v1)
        vv = transpose(vh)
        put(LL, LL, p_mul2(vv, vh)); put(LL, HL, p_mul2(vv, uh))
        put(LL, LH, p_mul2(uv, vh)); put(LL, HH, p_mul2(uv, uh))
        put(HL, LL, p_mul2(vv, ph)); put(HL, HL, vv)
        put(HL, LH, p_mul2(uv, ph)); put(HL, HH, uv)
        put(LH, LL, p_mul2(pv, vh)); put(LH, HL, p_mul2(pv, uh))
        put(LH, LH, vh); put(LH, HH, uh)
        put(HH, LL, p_mul2(pv, ph)); put(HH, HL, pv); put(HH, LH, ph)
    else:
        raise ValueError(kind)
    return m


def is_identity(m: dict) -> bool:
    for (i, j), p in m.items():
        if i == j and not is_one(p):
            return False
        if i != j and p:
            return False
    return True


def m_mul(a: dict, b: dict) -> dict:
    """Matrix product a*b (a acts after b), polyphase.cpp:173-183."""
    r = {}
    for i in range(4):
        for j in range(4):
            acc = {}
            for k in range(4):
                if (i, k) in a and (k, j) in b:
                    acc = p_add(acc, p_mul2(a[(i, k)], b[(k, j)]))
            if acc:
                r[(i, j)] = acc
    return r


# -------------------------------------------------------------------- schemes
@dataclass
class Step:
    label: str
    kind: str
    barrier: bool
    matrix: dict
    predict: dict = field(default_factory=dict)
    update: dict = field(default_factory=dict)


@dataclass
class Scheme:
    wavelet: Wavelet
    name: str
    steps: list
    conv: list | None = None    # [f_ll, f_hl, f_lh, f_hh] 2-D polys

    @property
    def barriers(self) -> int:
        """schemes.cpp:193-198 (Convolution charged the data barrier)."""
        if self.name == "convolution":
            return 1
        return sum(1 for s in self.steps if s.barrier)

    @property
    def macs(self) -> int:
        """schemes.cpp:176-191."""
        if self.name == "convolution":
            return sum(len(f) for f in self.conv)
        n = 0
        for s in self.steps:
            for (i, j), p in s.matrix.items():
                if i == j and is_one(p):
                    continue
                n += len(p)
        return n


def _push(steps, kind, p, u, barrier, label, one):
    m = build_matrix(kind, p, u, one)
    if is_identity(m):
        return  # schemes.cpp:43-44: degenerate steps are omitted
    steps.append(Step(label, kind, barrier, m, dict(p), dict(u)))


def _base_stage(steps, name, p, u, one):
    """schemes.cpp:49-81."""
    z = {}
    if name == "sweldens":
        _push(steps, "T_H", p, z, True, "T_H", one)
        _push(steps, "T_V", p, z, True, "T_V", one)
        _push(steps, "S_H", z, u, True, "S_H", one)
        _push(steps, "S_V", z, u, True, "S_V", one)
    elif name == "iwahashi":
        _push(steps, "T_I", p, z, True, "T_I", one)
        _push(steps, "R_I", p, u, True, "R_I", one)
        _push(steps, "S_I", z, u, True, "S_I", one)
    elif name == "explosive":
        _push(steps, "T_E", p, z, True, "T_E", one)
        _push(steps, "R_E", p, u, True, "R_E", one)
        _push(steps, "S_E", z, u, True, "S_E", one)
    elif name == "monolithic":
        _push(steps, "T_MONO", p, z, True, "T_P", one)
        _push(steps, "S_MONO", z, u, True, "S_U", one)
    elif name == "polyphase":
        _push(steps, "N_FULL", p, u, True, "N", one)
    else:
        raise ValueError(name)


def _star_stage(steps, name, p, u, one):
    """schemes.cpp:83-142."""
    p0, p1 = split_scalar(p)
    u0, u1 = split_scalar(u)
    base = name[:-len("_star")]
    if not p0 and not u0:
        _base_stage(steps, base, p, u, one)
        return
    z = {}
    if name in ("iwahashi_star", "explosive_star"):
        iwa = name == "iwahashi_star"
        _push(steps, "T_H", p0, z, False, "T_H(P0)", one)
        _push(steps, "T_V", p0, z, False, "T_V(P0)", one)
        _push(steps, "T_I" if iwa else "T_E", p1, z, True, "T_I(P1)" if iwa else "T_E(P1)", one)
        _push(steps, "R_I" if iwa else "R_E", p1, u1, True,
              "R_I(P1,U1)" if iwa else "R_E(P1,U1)", one)
        _push(steps, "S_I" if iwa else "S_E", z, u1, True, "S_I(U1)" if iwa else "S_E(U1)", one)
        _push(steps, "S_H", z, u0, False, "S_H(U0)", one)
        _push(steps, "S_V", z, u0, False, "S_V(U0)", one)
    elif name == "monolithic_star":
        _push(steps, "T_MONO", p1, z, True, "T_P(P1)", one)
        _push(steps, "T_H", p0, z, False, "T_H(P0)", one)
        _push(steps, "T_V", p0, z, False, "T_V(P0)", one)
        _push(steps, "S_MONO", z, u1, True, "S_U(U1)", one)
        _push(steps, "S_H", z, u0, False, "S_H(U0)", one)
        _push(steps, "S_V", z, u0, False, "S_V(U0)", one)
    elif name == "polyphase_star":
        _push(steps, "T_H", p0, z, False, "T_H(P0)", one)
        _push(steps, "T_V", p0, z, False, "T_V(P0)", one)
        _push(steps, "N_FULL", p1, u1, True, "N(P1,U1)", one)
        _push(steps, "S_H", z, u0, False, "S_H(U0)", one)
        _push(steps, "S_V", z, u0, False, "S_V(U0)", one)
    else:
        raise ValueError(name)


def analysis_filters(w: Wavelet):
    """wavelets.cpp:76-78 via polyphase.cpp:239-299: interleave the phases of
    the 1-D lifting product (scaling excluded) into (g0, g1)."""
    one = w.one
    # 2x2 over rows (L, H) x cols (E, O); acc = U P ... (first stage first)
    a, b, c, d = {0: one}, {}, {}, {0: one}
    for p, u in w.stages:
        # predict [[1,0],[P,1]] then update [[1,U],[0,1]]
        a, b, c, d = a, b, p_add(p_mul1(p, a), c), p_add(p_mul1(p, b), d)
        a, b, c, d = p_add(a, p_mul1(u, c)), p_add(b, p_mul1(u, d)), c, d
    g0o, g0e, g1o, g1e = b, a, c, d  # PolyMatrix2{acc.c, acc.d, acc.b, acc.a} naming
    # polyphase.cpp:297: m{g1o=acc.c, g1e=acc.d, g0o=acc.b, g0e=acc.a}
    g1o, g1e, g0o, g0e = c, d, b, a
    g0, g1 = {}, {}
    for e, v in g0e.items():
        g0[2 * e] = v
    for e, v in g0o.items():
        g0[2 * e - 1] = v
    for e, v in g1e.items():
        g1[2 * e] = v
    for e, v in g1o.items():
        g1[2 * e + 1] = v
    return _clean(g0), _clean(g1)


def conv2d_filters(w: Wavelet):
    """wavelets.cpp:80-88: F_ss' = g_s(z_n) g_s'(z_m)."""
    g0, g1 = analysis_filters(w)
    g0h, g1h = orient_h(g0), orient_h(g1)
    g0v, g1v = transpose(g0h), transpose(g1h)
    return [p_mul2(g0v, g0h), p_mul2(g0v, g1h), p_mul2(g1v, g0h), p_mul2(g1v, g1h)]


def build_scheme(scheme: str, wavelet: str | Wavelet) -> Scheme:
    """schemes.cpp:146-174."""
    w = get_wavelet(wavelet) if isinstance(wavelet, str) else wavelet
    if scheme not in SCHEMES:
        raise ValueError(f"unknown scheme: {scheme}")
    if scheme == "convolution":
        return Scheme(w, scheme, [], conv2d_filters(w))
    steps: list = []
    for p, u in w.stages:
        if scheme.endswith("_star"):
            _star_stage(steps, scheme, p, u, w.one)
        else:
            _base_stage(steps, scheme, p, u, w.one)
    return Scheme(w, scheme, steps)


# ------------------------------------------------------------------ inverses
def invert_step(step: Step, one) -> Step:
    """Exact inverse of one step (see module docstring)."""
    if step.kind == "N_FULL":
        # N(P,U) = S_V(U) S_H(U) T_V(P) T_H(P)  =>  N^-1 applies S_V(-U),
        # S_H(-U), T_V(-P), T_H(-P) in that order; fused into one matrix so
        # the inverse keeps the forward's single barrier.
        seq = []
        if step.update:
            nu = p_neg(step.update)
            seq += [build_matrix("S_V", {}, nu, one), build_matrix("S_H", {}, nu, one)]
        if step.predict:
            np_ = p_neg(step.predict)
            seq += [build_matrix("T_V", np_, {}, one), build_matrix("T_H", np_, {}, one)]
        acc = seq[0]
        for s in seq[1:]:
            acc = m_mul(s, acc)
        return Step(step.label + "^-1", "N_INV", step.barrier, acc)
    n = {}
    for (i, j), p in step.matrix.items():
        q = p_add(p, {(0, 0): -one}) if i == j else dict(p)
        if q:
            n[(i, j)] = q
    neg_n = {k: p_neg(p) for k, p in n.items()}
    inv = {(i, i): {(0, 0): one} for i in range(4)}
    term = {(i, i): {(0, 0): one} for i in range(4)}
    for _ in range(8):
        term = m_mul(neg_n, term)
        if not term:
            break
        for k, p in term.items():
            s = p_add(inv.get(k, {}), p)
            if s:
                inv[k] = s
            else:
                inv.pop(k, None)
    else:
        raise RuntimeError("non-unipotent step")
    return Step(step.label + "^-1", step.kind + "_INV", step.barrier, inv)


def inverse_steps(s: Scheme) -> list:
    """Reversed, inverted step list. The barrier flag moves with the step
    whose neighbour reads it guards, so the inverse has the forward's barrier
    count. Convolution has no lifting factorisation; its inverse is the
    reference's own (Sweldens) inverse."""
    src = s if s.name != "convolution" else build_scheme("sweldens", s.wavelet)
    return [invert_step(st, s.wavelet.one) for st in reversed(src.steps)]


# ------------------------------------------------------------ kernel layout
def reads_neighbours(m: dict) -> bool:
    return any(k != (0, 0) for p in m.values() for k in p)


def epochs(steps: list) -> tuple[list, list]:
    """Groups a step list into (pre_local_steps, [(nbr_step, [local...])]).

    Every step that reads a spatial neighbour opens a new epoch (its data
    must be published behind a barrier); purely local (0,0) steps join the
    current epoch. Local steps before the first neighbour step run right
    after the load (Polyphase*/Iwahashi*/Explosive* T_H(P0), T_V(P0))."""
    pre, eps = [], []
    for st in steps:
        if reads_neighbours(st.matrix):
            eps.append((st, []))
        elif eps:
            eps[-1][1].append(st)
        else:
            pre.append(st)
    return pre, eps


def halo(steps: list) -> tuple[int, int, int, int]:
    """Cells of each component that become invalid when the tile's outside is
    garbage, propagated through every step: returns the reach (left, right,
    up, down) in quads needed for exact outputs (cf. parsim required_halo,
    parsim.cpp:185-218)."""
    # valid margin per component per side; reading offset (dr, dc) at a cell
    # needs the source valid at cell+offset.
    inv = {d: [0] * 4 for d in ("l", "r", "u", "d")}
    for st in steps:
        new = {d: list(v) for d, v in inv.items()}
        for (i, j), p in st.matrix.items():
            for (km, kn) in p:
                dc, dr = -km, -kn
                new["l"][i] = max(new["l"][i], inv["l"][j] + max(0, -dc))
                new["r"][i] = max(new["r"][i], inv["r"][j] + max(0, dc))
                new["u"][i] = max(new["u"][i], inv["u"][j] + max(0, -dr))
                new["d"][i] = max(new["d"][i], inv["d"][j] + max(0, dr))
        inv = new
    return max(inv["l"]), max(inv["r"]), max(inv["u"]), max(inv["d"])


def scheme_to_json(s: Scheme) -> dict:
    """Same shape as the reference dump (tools/make_golden.py) for diffing."""
    def poly(p):
        return [[k[0], k[1], str(v) if isinstance(v, Fraction) else repr(v), float(v)]
                for k, v in sorted(p.items())]
    out = {"wavelet": s.wavelet.name, "scheme": s.name, "zeta": s.wavelet.zeta,
           "exact": int(s.wavelet.exact), "barriers": s.barriers, "macs": s.macs,
           "steps": [{"label": st.label, "barrier": int(st.barrier), "kind": st.kind,
                      "entries": [[i, j, poly(st.matrix[(i, j)])] for (i, j) in
                                  sorted(st.matrix) if st.matrix[(i, j)]]}
                     for st in s.steps]}
    if s.conv is not None:
        out["conv"] = [poly(f) for f in s.conv]
    return out
