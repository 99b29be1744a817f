"""TEST INFRASTRUCTURE -- CPU oracle for the 2-D lifting DWT hot path.

NOT the product. Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference`` arm) may import
this module, and only as the checker / the timed reference.

Two CPU implementations live here:

* :class:`RefLib` -- the UNMODIFIED reference library
  (``/root/reference/proj/src/*.cpp``) compiled by ``oracle/Makefile`` into
  ``oracle/_ref/libwavelift_ref.so`` with a repo-owned Boost shim. It is the
  ground truth: ``forward`` / ``inverse`` / ``multi_level_*`` / ``apply_step``
  (``transform.cpp:100-256``) and ``build_scheme`` (``schemes.cpp:146-174``).
* :class:`Oracle` -- a plain-C restatement (``oracle/wl_oracle.c``) of the
  same algorithm, driven by the reference's own step tables, which were dumped
  from ``build_scheme`` into ``tests/golden/schemes_ref.json`` by
  ``tools/make_golden.py``. It is pinned against :class:`RefLib` and the golden
  fixtures in ``tests/test_oracle.py``, so it can stand in where the ``_ref``
  build is unavailable.

Per-scheme inverse step lists (the reference's ``inverse`` is wavelet-only,
``transform.cpp:178-196``) are derived here from the dumped forward tables by
exact (cdf53: ``Fraction``) or float (cdf97) Laurent-matrix inversion, see
:func:`inverse_step_list`.
"""
from __future__ import annotations

import ctypes
import json
import os
from fractions import Fraction

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
GOLDEN = os.path.join(ROOT, "tests", "golden")

WAVELETS = ["cdf53", "cdf97", "dd137"]
SCHEMES = ["sweldens", "iwahashi", "iwahashi_star", "explosive", "explosive_star",
           "monolithic", "monolithic_star", "polyphase", "polyphase_star", "convolution"]
BOUNDARIES = ["periodic", "symmetric"]
LL, HL, LH, HH = 0, 1, 2, 3

_dbl_p = ctypes.POINTER(ctypes.c_double)
_int_p = ctypes.POINTER(ctypes.c_int)


def _ptr(a, kind=_dbl_p):
    return a.ctypes.data_as(kind)


def _idx(table, name):
    return table.index(name) if isinstance(name, str) else int(name)


# --------------------------------------------------------------------- tables
_SCHEME_CACHE: dict | None = None


def scheme_tables() -> dict:
    """The reference's build_scheme() output for every wavelet x scheme, as
    dumped from oracle/_ref (tests/golden/schemes_ref.json)."""
    global _SCHEME_CACHE
    if _SCHEME_CACHE is None:
        with open(os.path.join(GOLDEN, "schemes_ref.json")) as f:
            _SCHEME_CACHE = json.load(f)
    return _SCHEME_CACHE


def _coeff(term, exact):
    km, kn, s, d = term
    return Fraction(s) if exact else float(d)


def step_matrix(step: dict, exact: bool) -> dict:
    """{(dst, src): {(km, kn): coeff}} from a dumped step."""
    m = {}
    for r, c, terms in step["entries"]:
        m[(r, c)] = {(t[0], t[1]): _coeff(t, exact) for t in terms}
    return m


def _is_one(p):
    return len(p) == 1 and p.get((0, 0)) == 1


def _padd(a, b):
    r = dict(a)
    for k, v in b.items():
        r[k] = r.get(k, 0) + v
        if r[k] == 0:
            del r[k]
    return r


def _pmul(a, b):
    r = {}
    for (am, an), av in a.items():
        for (bm, bn), bv in b.items():
            k = (am + bm, an + bn)
            r[k] = r.get(k, 0) + av * bv
            if r[k] == 0:
                del r[k]
    return r


def _mmul(a, b):
    """(a b) for 4x4 Laurent matrices (a acts after b), polyphase.cpp:173-183."""
    r = {}
    for i in range(4):
        for j in range(4):
            acc = {}
            for k in range(4):
                if (i, k) in a and (k, j) in b:
                    acc = _padd(acc, _pmul(a[(i, k)], b[(k, j)]))
            if acc:
                r[(i, j)] = acc
    return r


def _identity(one):
    return {(i, i): {(0, 0): one} for i in range(4)}


def _separable(kind, op_h, neg=True):
    """T_H/T_V/S_H/S_V placements (polyphase.cpp:85-100) for a horizontal
    1-D operator given as {km: coeff} embedded as {(km, 0): c}."""
    one = next(iter(op_h.values())) * 0 + 1
    sign = -1 if neg else 1
    h = {k: sign * v for k, v in op_h.items()}
    v = {(k[1], k[0]): c for k, c in h.items()}
    m = _identity(one)
    if kind == "T_H":
        m[(HL, LL)] = h
        m[(HH, LH)] = h
    elif kind == "T_V":
        m[(LH, LL)] = v
        m[(HH, HL)] = v
    elif kind == "S_H":
        m[(LL, HL)] = h
        m[(LH, HH)] = h
    elif kind == "S_V":
        m[(LL, LH)] = v
        m[(HL, HH)] = v
    return m


def invert_step(m: dict, kind: str, one) -> dict:
    """Exact inverse of one step matrix.

    Unipotent kinds (every kind but N_FULL): M = I + N with N nilpotent, so
    M^-1 = I - N + N^2 - ... (terminates structurally). N_FULL(P, U) is the
    Sweldens product S_V S_H T_V T_H, whose inverse is the negated reversed
    product S_V(-U), S_H(-U), T_V(-P), T_H(-P) (transform.cpp:178-196,
    polyphase.cpp:147-167: P = entry(HH, LH), U = entry(LH, HH))."""
    if kind == "N_FULL":
        p = m.get((HH, LH), {})
        u = m.get((LH, HH), {})
        seq = []
        if u:
            seq += [_separable("S_V", u), _separable("S_H", u)]
        if p:
            seq += [_separable("T_V", p), _separable("T_H", p)]
        acc = seq[0]
        for s in seq[1:]:
            acc = _mmul(s, acc)
        return acc
    n = {}
    for (i, j), p in m.items():
        q = dict(p)
        if i == j:
            q = _padd(q, {(0, 0): -one})
        if q:
            n[(i, j)] = q
    neg_n = {k: {t: -c for t, c in p.items()} for k, p in n.items()}
    inv = _identity(one)
    term = _identity(one)
    for _ in range(8):
        term = _mmul(neg_n, term)
        if not term:
            break
        for k, p in term.items():
            s = _padd(inv.get(k, {}), p)
            if s:
                inv[k] = s
            elif k in inv:
                del inv[k]
    else:
        raise RuntimeError("step matrix is not unipotent")
    return inv


def inverse_step_list(wavelet: str, scheme: str) -> list[dict]:
    """Reversed list of inverted forward steps (each a {(dst, src): poly})."""
    t = scheme_tables()[wavelet][scheme]
    exact = bool(t["exact"])
    one = Fraction(1) if exact else 1.0
    return [invert_step(step_matrix(s, exact), s["kind"], one) for s in reversed(t["steps"])]


def reference_inverse_list(wavelet: str) -> list[dict]:
    """The reference inverse (transform.cpp:178-196): per stage, reversed,
    S_V(-U), S_H(-U), T_V(-P), T_H(-P) -- i.e. the sweldens inverse list."""
    return inverse_step_list(wavelet, "sweldens")


def flatten(steps: list[dict]):
    """Tap arrays in the reference summation order (transform.cpp:103-116)."""
    counts, taps, coeffs = [], [], []
    for m in steps:
        n0 = len(coeffs)
        for dst in range(4):
            for src in range(4):
                p = m.get((dst, src))
                if not p:
                    continue
                if dst == src and _is_one(p):
                    taps.append((dst, src, 0, 0, 1))
                    coeffs.append(1.0)
                    continue
                for (km, kn) in sorted(p):
                    taps.append((dst, src, km, kn, 0))
                    coeffs.append(float(p[(km, kn)]))
        counts.append(len(coeffs) - n0)
    return (np.asarray(counts, dtype=np.int32), np.asarray(taps, dtype=np.int32).reshape(-1, 5),
            np.asarray(coeffs, dtype=np.float64))


def forward_step_list(wavelet: str, scheme: str) -> list[dict]:
    t = scheme_tables()[wavelet][scheme]
    return [step_matrix(s, bool(t["exact"])) for s in t["steps"]]


# ---------------------------------------------------------------- C oracle
class Oracle:
    """Plain-C restatement (oracle/wl_oracle.c) of transform.cpp."""

    def __init__(self, path: str | None = None):
        path = path or os.path.join(HERE, "_build", "libwl_oracle.so")
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        lib = ctypes.CDLL(path)
        lib.wlo_resolve_index.restype = ctypes.c_int
        lib.wlo_resolve_index.argtypes = [ctypes.c_int] * 3
        self.lib = lib

    def resolve_index(self, i, n, boundary):
        return self.lib.wlo_resolve_index(i, n, _idx(BOUNDARIES, boundary))

    def _steps(self, steps):
        counts, taps, coeffs = flatten(steps)
        return counts, np.ascontiguousarray(taps), coeffs

    def apply_step(self, q4: np.ndarray, step: dict, boundary) -> np.ndarray:
        q4 = np.ascontiguousarray(q4, dtype=np.float64)
        _, qh, qw = q4.shape
        counts, taps, coeffs = self._steps([step])
        out = np.empty_like(q4)
        self.lib.wlo_apply_step(_ptr(q4), qw, qh, _ptr(taps, _int_p), _ptr(coeffs),
                                int(counts[0]), _idx(BOUNDARIES, boundary), _ptr(out))
        return out

    def forward(self, img, wavelet, scheme, boundary="periodic", scaling=False):
        img = np.ascontiguousarray(img, dtype=np.float64)
        h, w = img.shape
        if w <= 0 or h <= 0 or w % 2 or h % 2:
            raise ValueError("forward requires even positive dimensions")
        t = scheme_tables()[wavelet][scheme]
        out = np.empty((4, h // 2, w // 2), dtype=np.float64)
        b = _idx(BOUNDARIES, boundary)
        if scheme == "convolution":
            ntap, taps, coeffs = [], [], []
            for f in t["conv"]:
                ntap.append(len(f))
                for km, kn, s, d in f:
                    taps.append((km, kn))
                    coeffs.append(float(Fraction(s)) if t["exact"] else float(d))
            ntap = np.asarray(ntap, dtype=np.int32)
            taps = np.asarray(taps, dtype=np.int32).reshape(-1, 2)
            coeffs = np.asarray(coeffs, dtype=np.float64)
            self.lib.wlo_forward_conv(_ptr(img), w, h, _ptr(ntap, _int_p), _ptr(taps, _int_p),
                                      _ptr(coeffs), b, int(scaling), ctypes.c_double(t["zeta"]),
                                      _ptr(out))
            return out
        counts, taps, coeffs = self._steps(forward_step_list(wavelet, scheme))
        self.lib.wlo_forward_steps(_ptr(img), w, h, len(counts), _ptr(counts, _int_p),
                                   _ptr(taps, _int_p), _ptr(coeffs), b, int(scaling),
                                   ctypes.c_double(t["zeta"]), _ptr(out))
        return out

    def inverse(self, q4, wavelet, boundary="periodic", undo_scaling=False, scheme=None):
        """scheme=None is the reference's wavelet-only inverse (sweldens list);
        a scheme name selects that scheme's reversed inverted step list."""
        q4 = np.ascontiguousarray(q4, dtype=np.float64)
        _, qh, qw = q4.shape
        t = scheme_tables()[wavelet]["sweldens"]
        steps = inverse_step_list(wavelet, scheme if scheme not in (None, "convolution")
                                  else "sweldens")
        counts, taps, coeffs = self._steps(steps)
        img = np.empty((2 * qh, 2 * qw), dtype=np.float64)
        self.lib.wlo_inverse_steps(_ptr(q4), qw, qh, len(counts), _ptr(counts, _int_p),
                                   _ptr(taps, _int_p), _ptr(coeffs), _idx(BOUNDARIES, boundary),
                                   int(undo_scaling), ctypes.c_double(t["zeta"]), _ptr(img))
        return img

    def pyramid_forward(self, img, wavelet, scheme, levels, boundary="periodic", scaling=False):
        """Flat pyramid: per level (finest first) HL, LH, HH, then coarsest LL."""
        img = np.asarray(img, dtype=np.float64)
        h, w = img.shape
        if levels < 1 or w % (1 << levels) or h % (1 << levels):
            raise ValueError("bad pyramid levels")
        parts, cur = [], img
        for _ in range(levels):
            q = self.forward(cur, wavelet, scheme, boundary, scaling)
            parts.append(q[1:].ravel())
            cur = q[0]
        parts.append(cur.ravel())
        return np.concatenate(parts)

    def pyramid_inverse(self, flat, w, h, levels, wavelet, boundary="periodic",
                        undo_scaling=False, scheme=None):
        sizes, pw, ph = [], w // 2, h // 2
        for l in range(levels):
            sizes.append((pw, ph))
            if l + 1 < levels:
                pw, ph = pw // 2, ph // 2
        offs, off = [], 0
        for (a, b) in sizes:
            offs.append(off)
            off += 3 * a * b
        ll = np.asarray(flat[off:off + pw * ph]).reshape(ph, pw)
        for l in range(levels - 1, -1, -1):
            a, b = sizes[l]
            det = np.asarray(flat[offs[l]:offs[l] + 3 * a * b]).reshape(3, b, a)
            ll = self.inverse(np.concatenate([ll[None], det]), wavelet, boundary, undo_scaling,
                              scheme)
        return ll


# ---------------------------------------------------------------- reference
class RefLib:
    """ctypes view of oracle/_ref/libwavelift_ref.so (the unmodified reference)."""

    def __init__(self, path: str | None = None):
        path = path or os.path.join(HERE, "_ref", "libwavelift_ref.so")
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` where "
                                    "/root/reference exists")
        lib = ctypes.CDLL(path)
        lib.wlref_last_error.restype = ctypes.c_char_p
        lib.wlref_dump_scheme.restype = ctypes.c_long
        lib.wlref_dump_scheme.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_char_p,
                                          ctypes.c_long]
        lib.wlref_random_image.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint,
                                           ctypes.c_int, _dbl_p]
        self.lib = lib

    @staticmethod
    def available() -> bool:
        return os.path.exists(os.path.join(HERE, "_ref", "libwavelift_ref.so"))

    def _check(self, st):
        if st == 1:
            raise ValueError(self.lib.wlref_last_error().decode())
        if st != 0:
            raise RuntimeError(self.lib.wlref_last_error().decode())

    def worker_count(self):
        return self.lib.wlref_worker_count()

    def random_image(self, w, h, seed, dyadic=False):
        out = np.empty((h, w), dtype=np.float64)
        self.lib.wlref_random_image(w, h, seed, int(dyadic), _ptr(out))
        return out

    def dump_scheme(self, wavelet, scheme) -> dict:
        wi, si = _idx(WAVELETS, wavelet), _idx(SCHEMES, scheme)
        n = self.lib.wlref_dump_scheme(wi, si, None, 0)
        buf = ctypes.create_string_buffer(n + 1)
        self.lib.wlref_dump_scheme(wi, si, buf, n + 1)
        return json.loads(buf.value.decode())

    def cost(self, wavelet, scheme):
        b, m = ctypes.c_int(), ctypes.c_long()
        self._check(self.lib.wlref_cost(_idx(WAVELETS, wavelet), _idx(SCHEMES, scheme),
                                        ctypes.byref(b), ctypes.byref(m)))
        return b.value, m.value

    def verify_identity(self, wavelet, scheme):
        d, m = ctypes.c_double(), ctypes.c_int()
        self._check(self.lib.wlref_verify_identity(_idx(WAVELETS, wavelet),
                                                   _idx(SCHEMES, scheme), ctypes.byref(d),
                                                   ctypes.byref(m)))
        return bool(m.value), d.value

    def forward(self, img, wavelet, scheme, boundary="periodic", scaling=False):
        img = np.ascontiguousarray(img, dtype=np.float64)
        h, w = img.shape
        out = np.empty((4, max(h // 2, 0), max(w // 2, 0)), dtype=np.float64)
        self._check(self.lib.wlref_forward(_ptr(img), w, h, _idx(WAVELETS, wavelet),
                                           _idx(SCHEMES, scheme), _idx(BOUNDARIES, boundary),
                                           int(scaling), _ptr(out)))
        return out

    def inverse(self, q4, wavelet, boundary="periodic", undo_scaling=False):
        q4 = np.ascontiguousarray(q4, dtype=np.float64)
        _, qh, qw = q4.shape
        img = np.empty((2 * qh, 2 * qw), dtype=np.float64)
        self._check(self.lib.wlref_inverse(_ptr(q4), qw, qh, _idx(WAVELETS, wavelet),
                                           _idx(BOUNDARIES, boundary), int(undo_scaling),
                                           _ptr(img)))
        return img

    def apply_step(self, q4, step: dict, boundary="periodic"):
        q4 = np.ascontiguousarray(q4, dtype=np.float64)
        _, qh, qw = q4.shape
        taps, coeffs = [], []
        for (d, s), p in step.items():
            for (km, kn), c in p.items():
                taps.append((d, s, km, kn))
                coeffs.append(float(c))
        taps = np.asarray(taps, dtype=np.int32).reshape(-1, 4)
        coeffs = np.asarray(coeffs, dtype=np.float64)
        out = np.empty_like(q4)
        self._check(self.lib.wlref_apply_step(_ptr(q4), qw, qh, _ptr(taps, _int_p),
                                              _ptr(coeffs), len(coeffs),
                                              _idx(BOUNDARIES, boundary), _ptr(out)))
        return out

    def pyramid_forward(self, img, wavelet, scheme, levels, boundary="periodic", scaling=False):
        img = np.ascontiguousarray(img, dtype=np.float64)
        h, w = img.shape
        out = np.empty(h * w, dtype=np.float64)
        self._check(self.lib.wlref_pyramid_forward(_ptr(img), w, h, _idx(WAVELETS, wavelet),
                                                   _idx(SCHEMES, scheme), levels,
                                                   _idx(BOUNDARIES, boundary), int(scaling),
                                                   _ptr(out)))
        return out

    def pyramid_inverse(self, flat, w, h, levels, wavelet, boundary="periodic",
                        undo_scaling=False):
        flat = np.ascontiguousarray(flat, dtype=np.float64)
        img = np.empty((h, w), dtype=np.float64)
        self._check(self.lib.wlref_pyramid_inverse(_ptr(flat), w, h, levels,
                                                   _idx(WAVELETS, wavelet),
                                                   _idx(BOUNDARIES, boundary),
                                                   int(undo_scaling), _ptr(img)))
        return img
