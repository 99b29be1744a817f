"""wavelift_b200 -- B200-native 2-D lifting DWT (CDF 5/3, CDF 9/7; all schemes).

Python host side of the drop-in surface. It mirrors the reference's C++
transform API (``/root/reference/proj/include/wavelift/transform.hpp:14-95``,
``schemes.hpp:15-62``, ``wavelets.hpp:21-32``) over device ``torch`` tensors and
calls the CUDA kernels through the C-ABI in ``include/wl_dwt.h``
(``libwavelift_b200.so``, built in-tree for sm_100a). There is no CPU
fallback: without the library or a GPU every call raises.

Names follow the reference: ``get_wavelet``, ``build_scheme``,
``parse_scheme`` / ``scheme_name``, ``parse_boundary`` / ``boundary_name``,
``forward``, ``inverse``, ``multi_level_forward``, ``multi_level_inverse``,
``resolve_index``. Errors map to the reference's exception classes:
``ValueError`` for ``std::invalid_argument`` and ``RuntimeError`` otherwise.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

from .schemes import BOUNDARIES, SCHEMES, WAVELETS  # noqa: F401

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("WL_LIB") or os.path.join(_PKG, "libwavelift_b200.so")

WL_OK, WL_EINVAL, WL_ERUNTIME = 0, 1, 2
ENGINE_AUTO, ENGINE_INTERP, ENGINE_FAST = 0, 1, 2

_lib = None


def lib() -> ctypes.CDLL:
    """Loads libwavelift_b200.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing -- run __graft_entry__.build() "
                               "(no CPU fallback exists)")
        l = ctypes.CDLL(LIB_PATH)
        vp, i, lg, fp = ctypes.c_void_p, ctypes.c_int, ctypes.c_long, ctypes.c_void_p
        l.wl_last_error.restype = ctypes.c_char_p
        l.wl_version.restype = ctypes.c_char_p
        l.wl_scheme_info.argtypes = [i, i, i, ctypes.POINTER(i), ctypes.POINTER(lg),
                                     ctypes.POINTER(i), ctypes.POINTER(i)]
        l.wl_resolve_index.argtypes = [i, i, i]
        l.wl_dwt2_forward.argtypes = [fp, i, i, lg, i, i, i, i, fp, fp, fp, fp, lg, vp]
        l.wl_dwt2_inverse.argtypes = [fp, fp, fp, fp, i, i, lg, i, i, i, i, fp, lg, vp]
        l.wl_pyramid_elems.restype = ctypes.c_size_t
        l.wl_pyramid_elems.argtypes = [i, i, i]
        l.wl_pyramid_scratch_elems.restype = ctypes.c_size_t
        l.wl_pyramid_scratch_elems.argtypes = [i, i, i]
        l.wl_dwt2_pyramid_forward.argtypes = [fp, i, i, i, i, i, i, i, fp, fp, vp]
        l.wl_dwt2_pyramid_inverse.argtypes = [fp, i, i, i, i, i, i, i, fp, fp, vp]
        l.wl_dwt2_forward_batch.argtypes = [fp, i, i, lg, lg, i, i, i, i, i, fp, fp, fp, fp,
                                            lg, lg, vp]
        l.wl_dwt2_inverse_batch.argtypes = [fp, fp, fp, fp, i, i, lg, lg, i, i, i, i, i, fp,
                                            lg, lg, vp]
        l.wl_pyramid_batch_scratch_elems.restype = ctypes.c_size_t
        l.wl_pyramid_batch_scratch_elems.argtypes = [i, i, i, i]
        l.wl_dwt2_pyramid_forward_batch.argtypes = [fp, i, i, lg, i, i, i, i, i, i, fp, lg, fp,
                                                    vp]
        l.wl_dwt2_pyramid_inverse_batch.argtypes = [fp, i, i, lg, i, i, i, i, i, i, fp, lg, fp,
                                                    vp]
        l.wl_strip_halo_rows.argtypes = [i, i, i]
        l.wl_dwt2_forward_strip.argtypes = [fp, i, i, i, lg, i, i, i, fp, fp, fp, fp, lg, vp]
        l.wl_dwt2_inverse_strip.argtypes = [fp, fp, fp, fp, i, i, i, lg, i, i, i, fp, lg, vp]
        l.wl_strips_last_error.restype = ctypes.c_char_p
        l.wl_strips_blob_bytes.restype = ctypes.c_size_t
        l.wl_strips_create.argtypes = [i, i, i, i, i, i, i, i, ctypes.POINTER(vp)]
        l.wl_strips_export.argtypes = [vp, ctypes.c_char_p]
        l.wl_strips_connect.argtypes = [vp, ctypes.c_char_p, ctypes.c_char_p]
        l.wl_strips_input.restype = vp
        l.wl_strips_input.argtypes = [vp]
        l.wl_strips_slice_elems.restype = ctypes.c_size_t
        l.wl_strips_slice_elems.argtypes = [vp]
        l.wl_strips_forward.argtypes = [vp, fp, vp]
        l.wl_strips_create_ex.argtypes = [i, i, i, i, i, i, i, i, i, ctypes.POINTER(vp)]
        l.wl_strips_inverse.argtypes = [vp, fp, fp, vp]
        l.wl_strips_check.argtypes = [vp]
        l.wl_strips_destroy.argtypes = [vp]
        l.wl_dwt2_forward_host.argtypes = [fp, i, i, lg, i, i, i, i, fp, fp, fp, fp, lg]
        l.wl_dwt2_inverse_host.argtypes = [fp, fp, fp, fp, i, i, lg, i, i, i, i, fp, lg]
        l.wl_set_engine.argtypes = [i]
        l.wl_launch_count.restype = lg
        if hasattr(l, "wl_set_graphs"):
            l.wl_set_graphs.argtypes = [i]
        ip, dp = ctypes.POINTER(i), ctypes.POINTER(ctypes.c_double)
        l.wl_scheme_nsteps.argtypes = [i, i]
        l.wl_scheme_step.argtypes = [i, i, i, ip, ip, ip, ctypes.c_char_p, i]
        l.wl_scheme_step_terms.argtypes = [i, i, i, ip, ip, ip, ip, dp, i]
        l.wl_scheme_conv_filter.argtypes = [i, i, ip, ip, dp, i]
        l.wl_apply_step.argtypes = [fp, fp, fp, fp, i, i, lg, i, ip, ip, ip, ip, dp, i, fp, fp,
                                    fp, fp, lg, vp]
        _lib = l
    return _lib


def _check(status: int):
    if status == WL_OK:
        return
    msg = lib().wl_last_error().decode()
    if status == WL_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(msg)


def version() -> str:
    return lib().wl_version().decode()


def set_engine(engine: int) -> int:
    """0 auto, 1 generic tile interpreter, 2 fast register-tile engine."""
    return lib().wl_set_engine(engine)


def set_graphs(on: bool) -> bool:
    """Graph replay of repeated pyramid calls (wl_set_graphs); returns the
    previous setting."""
    return bool(lib().wl_set_graphs(int(bool(on))))


def launch_count() -> int:
    return lib().wl_launch_count()


# ---------------------------------------------------------------- selection
def _index(table, name, what):
    if isinstance(name, int):
        if 0 <= name < len(table):
            return name
    elif name in table:
        return table.index(name)
    raise ValueError(f"unknown {what}: {name}")


def scheme_name(kind) -> str:
    """schemes.cpp:17-31."""
    return SCHEMES[_index(SCHEMES, kind, "scheme")]


def parse_scheme(name: str):
    """schemes.cpp:33-37: None for unknown names."""
    return SCHEMES.index(name) if name in SCHEMES else None


def boundary_name(mode) -> str:
    return BOUNDARIES[_index(BOUNDARIES, mode, "boundary")]


def parse_boundary(name: str):
    return BOUNDARIES.index(name) if name in BOUNDARIES else None


@dataclass(frozen=True)
class WaveletSpec:
    """wavelets.hpp:21-27 (constants live in the kernels' generated tables)."""
    name: str
    index: int
    zeta: float


def get_wavelet(name: str) -> WaveletSpec:
    """wavelets.cpp:27-62; ValueError for unknown names."""
    from .schemes import get_wavelet as _gw
    w = _gw(name)
    return WaveletSpec(w.name, WAVELETS.index(w.name), w.zeta)


MATRIX_KINDS = ("T_H", "T_V", "S_H", "S_V", "T_I", "R_I", "S_I", "T_E", "R_E", "S_E",
                "T_MONO", "S_MONO", "N_FULL")  # polyphase.hpp:24-38 MatrixKind


@dataclass(frozen=True)
class StepMatrix:
    """polyphase.hpp:45-68: 4x4 Laurent matrix over [LL, HL, LH, HH];
    entries[(row, col)] = {(k_m, k_n): coefficient} (double)."""
    entries: dict
    kind: str = "N_FULL"
    needs_barrier: bool = True

    def entry(self, row: int, col: int) -> dict:
        return self.entries.get((row, col), {})

    def is_identity(self) -> bool:
        return all((r == c and p == {(0, 0): 1.0}) or (r != c and not p)
                   for (r, c), p in self.entries.items()) and \
            all(self.entries.get((k, k)) == {(0, 0): 1.0} for k in range(4))


@dataclass(frozen=True)
class Step:
    """schemes.hpp:34-38."""
    matrix: StepMatrix
    needs_barrier: bool
    label: str


@dataclass(frozen=True)
class Scheme:
    """schemes.hpp:40-45: kind + wavelet; `steps` / `conv_filters` are read
    from the library's build_scheme tables (schemes.cpp:146-174)."""
    kind: int
    wavelet: WaveletSpec

    @property
    def name(self) -> str:
        return SCHEMES[self.kind]

    @property
    def steps(self) -> list:
        """The step sequence (empty for Convolution)."""
        l, w = lib(), self.wavelet.index
        n = l.wl_scheme_nsteps(w, self.kind)
        if n < 0:
            _check(WL_EINVAL)
        out = []
        for k in range(n):
            mk, nb, nt = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
            label = ctypes.create_string_buffer(64)
            _check(l.wl_scheme_step(w, self.kind, k, ctypes.byref(mk), ctypes.byref(nb),
                                    ctypes.byref(nt), label, 64))
            rows, cols, km, kn = [(ctypes.c_int * nt.value)() for _ in range(4)]
            co = (ctypes.c_double * nt.value)()
            l.wl_scheme_step_terms(w, self.kind, k, rows, cols, km, kn, co, nt.value)
            ent = {}
            for t in range(nt.value):
                ent.setdefault((rows[t], cols[t]), {})[(km[t], kn[t])] = co[t]
            out.append(Step(StepMatrix(ent, MATRIX_KINDS[mk.value], bool(nb.value)),
                            bool(nb.value), label.value.decode()))
        return out

    @property
    def conv_filters(self):
        """(f_ll, f_hl, f_lh, f_hh) as {(k_m, k_n): c} (Convolution only, else None)."""
        if SCHEMES[self.kind] != "convolution":
            return None
        l, out = lib(), []
        for f in range(4):
            n = l.wl_scheme_conv_filter(self.wavelet.index, f, None, None, None, 0)
            km, kn = (ctypes.c_int * n)(), (ctypes.c_int * n)()
            co = (ctypes.c_double * n)()
            l.wl_scheme_conv_filter(self.wavelet.index, f, km, kn, co, n)
            out.append({(km[t], kn[t]): co[t] for t in range(n)})
        return tuple(out)

    def info(self, direction: int = 0) -> dict:
        b, m, e, h = ctypes.c_int(), ctypes.c_long(), ctypes.c_int(), ctypes.c_int()
        _check(lib().wl_scheme_info(self.wavelet.index, self.kind, direction, ctypes.byref(b),
                                    ctypes.byref(m), ctypes.byref(e), ctypes.byref(h)))
        return {"barriers": b.value, "macs": m.value, "epochs": e.value, "halo": h.value}


def build_scheme(kind, wavelet) -> Scheme:
    """schemes.cpp:146-174 (selection only)."""
    w = wavelet if isinstance(wavelet, WaveletSpec) else get_wavelet(wavelet)
    return Scheme(_index(SCHEMES, kind, "scheme"), w)


def conv_polyphase_matrix(filters) -> StepMatrix:
    """polyphase.cpp:301-340: the polyphase reassembly of the four 2-D
    analysis filters into one 4x4 matrix."""
    ent = {}
    for target, f in enumerate(filters):
        col_high, row_high = target in (1, 3), target in (2, 3)
        for (km, kn), c in f.items():
            if not col_high:
                codd = km % 2 != 0
                a = (km + 1) // 2 if codd else km // 2
            else:
                codd = km % 2 == 0
                a = km // 2 if codd else (km - 1) // 2
            if not row_high:
                rodd = kn % 2 != 0
                b = (kn + 1) // 2 if rodd else kn // 2
            else:
                rodd = kn % 2 == 0
                b = kn // 2 if rodd else (kn - 1) // 2
            src = (2 if rodd else 0) + (1 if codd else 0)
            e = ent.setdefault((target, src), {})
            e[(a, b)] = e.get((a, b), 0.0) + c
    return StepMatrix(ent, "N_FULL", True)


def scheme_step_matrices(s: Scheme) -> list:
    """schemes.cpp:221-228: the scheme's own matrices, or the polyphase
    reassembly of the four filters for Convolution."""
    if SCHEMES[s.kind] == "convolution":
        return [conv_polyphase_matrix(s.conv_filters)]
    return [st.matrix for st in s.steps]


def apply_step(q, step, boundary="periodic", out=None, stream=None):
    """transform.cpp:100-125 on the GPU: out-of-place y_i = sum_j M_ij (*) x_j
    for a (4, qh, qw) float32 CUDA tensor; `step` is a Step or StepMatrix.
    Terms are summed in the reference's order (destination, source, then
    exponent map order), multiply and add unfused."""
    import torch
    q = _dev_f32(q, "q").contiguous()
    if q.dim() != 3 or q.shape[0] != 4:
        raise ValueError("q must be (4, qh, qw)")
    m = step.matrix if isinstance(step, Step) else step
    rows, cols, km, kn, co = [], [], [], [], []
    for (r, c) in sorted(m.entries):
        for (a, b) in sorted(m.entries[(r, c)]):
            rows.append(r)
            cols.append(c)
            km.append(a)
            kn.append(b)
            co.append(float(m.entries[(r, c)][(a, b)]))
    n = len(co)
    arr = lambda t, v: (t * max(n, 1))(*v)  # noqa: E731
    _, qh, qw = q.shape
    if out is None:
        out = torch.empty_like(q)
    _check(lib().wl_apply_step(q[0].data_ptr(), q[1].data_ptr(), q[2].data_ptr(),
                               q[3].data_ptr(), qw, qh, qw, n, arr(ctypes.c_int, rows),
                               arr(ctypes.c_int, cols), arr(ctypes.c_int, km),
                               arr(ctypes.c_int, kn), arr(ctypes.c_double, co),
                               _index(BOUNDARIES, boundary, "boundary"), out[0].data_ptr(),
                               out[1].data_ptr(), out[2].data_ptr(), out[3].data_ptr(),
                               out.stride(1), _stream_ptr(stream)))
    return out


def count_barriers(s: Scheme) -> int:
    return s.info()["barriers"]


def count_macs(s: Scheme) -> int:
    return s.info()["macs"]


def resolve_index(i: int, n: int, boundary) -> int:
    return lib().wl_resolve_index(i, n, _index(BOUNDARIES, boundary, "boundary"))


# ----------------------------------------------------------------- transforms
def _stream_ptr(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _dev_f32(t, what):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float32:
        raise ValueError(f"{what} must be a float32 CUDA tensor")
    return t


def _pitched(t):
    """(ptr, rows, cols, pitch) for a 2-D tensor with unit column stride."""
    if t.dim() != 2 or t.stride(1) != 1:
        t = t.contiguous()
    return t, t.stride(0)


def forward(img, scheme: Scheme, boundary="periodic", apply_scaling=False, out=None,
            stream=None):
    """transform.cpp:163-176: (h, w) float32 CUDA image -> (4, h/2, w/2) planes
    [LL, HL, LH, HH]."""
    import torch
    img = _dev_f32(img, "img")
    if img.dim() != 2:
        raise ValueError("img must be 2-D (height, width)")
    img, pitch = _pitched(img)
    h, w = img.shape
    if out is None:
        out = torch.empty((4, max(h // 2, 0), max(w // 2, 0)), device=img.device,
                          dtype=torch.float32)
    b = _index(BOUNDARIES, boundary, "boundary")
    p = [out[c].data_ptr() for c in range(4)]
    _check(lib().wl_dwt2_forward(img.data_ptr(), w, h, pitch, scheme.wavelet.index, scheme.kind,
                                 b, int(bool(apply_scaling)), p[0], p[1], p[2], p[3],
                                 out.stride(1) if out.dim() == 3 else w // 2,
                                 _stream_ptr(stream)))
    return out


def inverse(q, wavelet, boundary="periodic", undo_scaling=False, scheme=None, out=None,
            stream=None):
    """transform.cpp:178-196. `q` is (4, qh, qw). `scheme` picks the inverse
    kernel (default: the reference's separable/Sweldens inverse)."""
    import torch
    q = _dev_f32(q, "q").contiguous()
    if q.dim() != 3 or q.shape[0] != 4:
        raise ValueError("q must be (4, qh, qw)")
    w = wavelet if isinstance(wavelet, WaveletSpec) else get_wavelet(wavelet)
    kind = 0 if scheme is None else (scheme.kind if isinstance(scheme, Scheme)
                                     else _index(SCHEMES, scheme, "scheme"))
    _, qh, qw = q.shape
    if out is None:
        out = torch.empty((2 * qh, 2 * qw), device=q.device, dtype=torch.float32)
    b = _index(BOUNDARIES, boundary, "boundary")
    _check(lib().wl_dwt2_inverse(q[0].data_ptr(), q[1].data_ptr(), q[2].data_ptr(),
                                 q[3].data_ptr(), qw, qh, qw, w.index, kind, b,
                                 int(bool(undo_scaling)), out.data_ptr(), out.stride(0),
                                 _stream_ptr(stream)))
    return out


@dataclass
class Pyramid:
    """transform.hpp:74-83 over one flat device buffer: details finest first
    (hl, lh, hh views per level) and the coarsest ll view."""
    flat: object
    width: int
    height: int
    levels: int

    def level(self, l):
        w, h = self.width >> (l + 1), self.height >> (l + 1)
        off = sum(3 * (self.width >> (k + 1)) * (self.height >> (k + 1)) for k in range(l))
        n = w * h
        return tuple(self.flat[off + i * n: off + (i + 1) * n].view(h, w) for i in range(3))

    @property
    def ll(self):
        w, h = self.width >> self.levels, self.height >> self.levels
        return self.flat[self.flat.numel() - w * h:].view(h, w)


def multi_level_forward(img, scheme: Scheme, levels: int, boundary="periodic",
                        apply_scaling=False, stream=None, out=None, scratch=None) -> Pyramid:
    """transform.cpp:198-227. `out` (flat, w*h floats) and `scratch` may be
    passed to reuse buffers (repeated calls with the same buffers replay a
    CUDA graph, see set_graphs)."""
    import torch
    img = _dev_f32(img, "img").contiguous()
    h, w = img.shape
    n = lib().wl_pyramid_elems(w, h, levels)
    flat = out if out is not None else torch.empty(max(n, 1), device=img.device,
                                                   dtype=torch.float32)
    if out is not None and (_dev_f32(out, "out").numel() < n or not out.is_contiguous()):
        raise ValueError("out must be a contiguous float32 CUDA tensor of w*h elements")
    need = lib().wl_pyramid_scratch_elems(w, h, levels)
    if scratch is None or scratch.numel() < need:
        scratch = torch.empty(max(need, 1), device=img.device, dtype=torch.float32)
    _check(lib().wl_dwt2_pyramid_forward(img.data_ptr(), w, h, levels, scheme.wavelet.index,
                                         scheme.kind, _index(BOUNDARIES, boundary, "boundary"),
                                         int(bool(apply_scaling)), flat.data_ptr(),
                                         scratch.data_ptr(), _stream_ptr(stream)))
    return Pyramid(flat, w, h, levels)


def multi_level_inverse(pyr: Pyramid, wavelet, boundary="periodic", undo_scaling=False,
                        scheme=None, stream=None, out=None, scratch=None):
    """transform.cpp:229-256 (`out` / `scratch` reusable as in
    multi_level_forward)."""
    import torch
    w = wavelet if isinstance(wavelet, WaveletSpec) else get_wavelet(wavelet)
    kind = 0 if scheme is None else (scheme.kind if isinstance(scheme, Scheme)
                                     else _index(SCHEMES, scheme, "scheme"))
    flat = _dev_f32(pyr.flat, "pyramid").contiguous()
    if flat.numel() != pyr.width * pyr.height:
        raise ValueError("pyramid detail plane size does not match its level")
    if out is None:
        out = torch.empty((pyr.height, pyr.width), device=flat.device, dtype=torch.float32)
    need = lib().wl_pyramid_scratch_elems(pyr.width, pyr.height, pyr.levels)
    if scratch is None or scratch.numel() < need:
        scratch = torch.empty(max(need, 1), device=flat.device, dtype=torch.float32)
    _check(lib().wl_dwt2_pyramid_inverse(flat.data_ptr(), pyr.width, pyr.height, pyr.levels,
                                         w.index, kind, _index(BOUNDARIES, boundary, "boundary"),
                                         int(bool(undo_scaling)), out.data_ptr(),
                                         scratch.data_ptr(), _stream_ptr(stream)))
    return out


# ------------------------------------------------------------ batches (C5)
def _kind(scheme):
    if scheme is None:
        return 0
    return scheme.kind if isinstance(scheme, Scheme) else _index(SCHEMES, scheme, "scheme")


def forward_batch(imgs, scheme: Scheme, boundary="periodic", apply_scaling=False, out=None,
                  stream=None):
    """`forward` over a batch: (n, h, w) -> (n, 4, h/2, w/2), one launch."""
    import torch
    imgs = _dev_f32(imgs, "imgs").contiguous()
    if imgs.dim() != 3:
        raise ValueError("imgs must be (n, height, width)")
    n, h, w = imgs.shape
    if out is None:
        out = torch.empty((n, 4, max(h // 2, 0), max(w // 2, 0)), device=imgs.device,
                          dtype=torch.float32)
    b = _index(BOUNDARIES, boundary, "boundary")
    _check(lib().wl_dwt2_forward_batch(
        imgs.data_ptr(), w, h, w, h * w, n, scheme.wavelet.index, scheme.kind, b,
        int(bool(apply_scaling)), out[:, 0].data_ptr(), out[:, 1].data_ptr(),
        out[:, 2].data_ptr(), out[:, 3].data_ptr(), out.stride(2), out.stride(0),
        _stream_ptr(stream)))
    return out


def inverse_batch(q, wavelet, boundary="periodic", undo_scaling=False, scheme=None, out=None,
                  stream=None):
    """`inverse` over a batch: (n, 4, qh, qw) -> (n, 2qh, 2qw), one launch."""
    import torch
    q = _dev_f32(q, "q").contiguous()
    if q.dim() != 4 or q.shape[1] != 4:
        raise ValueError("q must be (n, 4, qh, qw)")
    w = wavelet if isinstance(wavelet, WaveletSpec) else get_wavelet(wavelet)
    n, _, qh, qw = q.shape
    if out is None:
        out = torch.empty((n, 2 * qh, 2 * qw), device=q.device, dtype=torch.float32)
    b = _index(BOUNDARIES, boundary, "boundary")
    _check(lib().wl_dwt2_inverse_batch(
        q[:, 0].data_ptr(), q[:, 1].data_ptr(), q[:, 2].data_ptr(), q[:, 3].data_ptr(), qw, qh,
        qw, q.stride(0), n, w.index, _kind(scheme), b, int(bool(undo_scaling)), out.data_ptr(),
        2 * qw, out.stride(0), _stream_ptr(stream)))
    return out


def multi_level_forward_batch(imgs, scheme: Scheme, levels: int, boundary="periodic",
                              apply_scaling=False, out=None, scratch=None, stream=None):
    """`multi_level_forward` over a batch (n, h, w): returns (n, h*w) flat
    pyramids (Pyramid layout per row); one launch per level."""
    import torch
    imgs = _dev_f32(imgs, "imgs").contiguous()
    if imgs.dim() != 3:
        raise ValueError("imgs must be (n, height, width)")
    n, h, w = imgs.shape
    if out is None:
        out = torch.empty((n, h * w), device=imgs.device, dtype=torch.float32)
    need = lib().wl_pyramid_batch_scratch_elems(w, h, levels, n)
    if scratch is None or scratch.numel() < need:
        scratch = torch.empty(max(need, 1), device=imgs.device, dtype=torch.float32)
    _check(lib().wl_dwt2_pyramid_forward_batch(
        imgs.data_ptr(), w, h, h * w, n, levels, scheme.wavelet.index, scheme.kind,
        _index(BOUNDARIES, boundary, "boundary"), int(bool(apply_scaling)), out.data_ptr(),
        out.stride(0), scratch.data_ptr(), _stream_ptr(stream)))
    return out


def multi_level_inverse_batch(pyrs, width, height, levels, wavelet, boundary="periodic",
                              undo_scaling=False, scheme=None, out=None, scratch=None,
                              stream=None):
    """`multi_level_inverse` over a batch of flat pyramids (n, h*w)."""
    import torch
    pyrs = _dev_f32(pyrs, "pyramids").contiguous()
    n = pyrs.shape[0]
    if pyrs.dim() != 2 or pyrs.shape[1] != width * height:
        raise ValueError("pyramid detail plane size does not match its level")
    w = wavelet if isinstance(wavelet, WaveletSpec) else get_wavelet(wavelet)
    if out is None:
        out = torch.empty((n, height, width), device=pyrs.device, dtype=torch.float32)
    need = lib().wl_pyramid_batch_scratch_elems(width, height, levels, n)
    if scratch is None or scratch.numel() < need:
        scratch = torch.empty(max(need, 1), device=pyrs.device, dtype=torch.float32)
    _check(lib().wl_dwt2_pyramid_inverse_batch(
        pyrs.data_ptr(), width, height, pyrs.stride(0), n, levels, w.index, _kind(scheme),
        _index(BOUNDARIES, boundary, "boundary"), int(bool(undo_scaling)), out.data_ptr(),
        out.stride(0), scratch.data_ptr(), _stream_ptr(stream)))
    return out


# ------------------------------------------------------- row strips (C4)
def strip_halo_rows(wavelet, scheme="monolithic_star", direction=0) -> int:
    """Halo (pixel rows for the forward, plane rows for the inverse) a strip
    transform needs on each side."""
    w = wavelet if isinstance(wavelet, WaveletSpec) else get_wavelet(wavelet)
    r = lib().wl_strip_halo_rows(w.index, _kind(scheme), direction)
    if r < 0:
        raise ValueError("strip transforms support cdf53/cdf97")
    return r


def forward_strip(buf, halo_rows: int, scheme: Scheme, apply_scaling=False, out=None,
                  stream=None):
    """Forward transform of the interior rows of a row strip.

    `buf` is (halo + rows + halo, w): the strip's own rows plus `halo_rows`
    rows of the neighbouring strips above and below (periodic image). The
    result (4, rows/2, w/2) equals the matching rows of `forward` of the whole
    image, bit for bit."""
    import torch
    buf = _dev_f32(buf, "buf")
    if buf.dim() != 2 or buf.stride(1) != 1:
        raise ValueError("buf must be a row-major 2-D tensor")
    rows = buf.shape[0] - 2 * halo_rows
    w = buf.shape[1]
    if out is None:
        out = torch.empty((4, max(rows // 2, 0), w // 2), device=buf.device, dtype=torch.float32)
    interior = buf[halo_rows:]
    _check(lib().wl_dwt2_forward_strip(
        interior.data_ptr(), w, rows, halo_rows, buf.stride(0), scheme.wavelet.index, scheme.kind,
        int(bool(apply_scaling)), out[0].data_ptr(), out[1].data_ptr(), out[2].data_ptr(),
        out[3].data_ptr(), out.stride(1), _stream_ptr(stream)))
    return out


def inverse_strip(q, halo_rows: int, wavelet, undo_scaling=False, scheme=None, out=None,
                  stream=None):
    """Inverse of a strip of planes `q` (4, halo + qrows + halo, qw) -> image
    rows (2*qrows, 2*qw)."""
    import torch
    q = _dev_f32(q, "q").contiguous()
    if q.dim() != 3 or q.shape[0] != 4:
        raise ValueError("q must be (4, rows, qw)")
    w = wavelet if isinstance(wavelet, WaveletSpec) else get_wavelet(wavelet)
    qrows = q.shape[1] - 2 * halo_rows
    qw = q.shape[2]
    if out is None:
        out = torch.empty((2 * max(qrows, 0), 2 * qw), device=q.device, dtype=torch.float32)
    p = [q[c, halo_rows:].data_ptr() for c in range(4)]
    _check(lib().wl_dwt2_inverse_strip(p[0], p[1], p[2], p[3], qw, qrows, halo_rows, qw,
                                       w.index, _kind(scheme), int(bool(undo_scaling)),
                                       out.data_ptr(), out.stride(0), _stream_ptr(stream)))
    return out


class _DevView:
    """__cuda_array_interface__ over a raw device pointer (zero-copy view)."""

    def __init__(self, ptr, shape):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f4",
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None}


def _scheck(status: int):
    if status == WL_OK:
        return
    msg = lib().wl_strips_last_error().decode()
    raise (ValueError if status == WL_EINVAL else RuntimeError)(msg)


class StripPyramid:
    """One rank's share of a row-strip multi-level pyramid (configs[3]).

    Rank `rank` of `nranks` owns image rows [rank*h/nranks, (rank+1)*h/nranks)
    of an h x w image (periodic: a ring; symmetric: ranks 0 and nranks-1 sit
    on the image edges). Levels exchange halo rows with the neighbour ranks
    through peer memory (CUDA IPC), see include/wl_dwt.h.
    Usage: `export()` -> share blobs -> `connect(up, down)` -> write
    `input` -> `forward()` / `inverse(slice)` (collective: every rank calls
    them equally often, in the same order)."""

    def __init__(self, w, h, levels, scheme: Scheme, rank=0, nranks=1, apply_scaling=False,
                 boundary="periodic"):
        self.w, self.h, self.levels = w, h, levels
        self.rank, self.nranks = rank, nranks
        self.rows = h // nranks if nranks > 0 else 0
        self.scheme = scheme
        self._ctx = ctypes.c_void_p()
        _scheck(lib().wl_strips_create_ex(w, h, rank, nranks, levels, scheme.wavelet.index,
                                          scheme.kind, _index(BOUNDARIES, boundary, "boundary"),
                                          int(bool(apply_scaling)), ctypes.byref(self._ctx)))
        import torch
        self.input = torch.as_tensor(_DevView(lib().wl_strips_input(self._ctx),
                                              (self.rows, w)), device="cuda")
        if nranks == 1:
            b = self.export()
            self.connect(b, b)

    def export(self) -> bytes:
        buf = ctypes.create_string_buffer(lib().wl_strips_blob_bytes())
        _scheck(lib().wl_strips_export(self._ctx, buf))
        return buf.raw

    def connect(self, up: bytes, down: bytes):
        _scheck(lib().wl_strips_connect(self._ctx, up, down))

    def slice_elems(self) -> int:
        return lib().wl_strips_slice_elems(self._ctx)

    def forward(self, out=None, stream=None):
        import torch
        if out is None:
            out = torch.empty(self.slice_elems(), device="cuda", dtype=torch.float32)
        _scheck(lib().wl_strips_forward(self._ctx, out.data_ptr(), _stream_ptr(stream)))
        return out

    def inverse(self, slice_, out=None, stream=None):
        """multi_level_inverse of this rank's slice -> its (rows, w) image rows."""
        import torch
        slice_ = _dev_f32(slice_, "slice").contiguous()
        if slice_.numel() != self.slice_elems():
            raise ValueError("slice size does not match this rank's pyramid slice")
        if out is None:
            out = torch.empty((self.rows, self.w), device="cuda", dtype=torch.float32)
        _scheck(lib().wl_strips_inverse(self._ctx, slice_.data_ptr(), out.data_ptr(),
                                        _stream_ptr(stream)))
        return out

    def check(self):
        _scheck(lib().wl_strips_check(self._ctx))

    def close(self):
        if self._ctx:
            lib().wl_strips_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def strip_slice_planes(slice_, w, rows, levels):
    """Views of a rank's pyramid slice: [(hl, lh, hh) per level], ll."""
    out, off = [], 0
    for l in range(levels):
        qw, qr = w >> (l + 1), rows >> (l + 1)
        n = qw * qr
        out.append(tuple(slice_[off + i * n: off + (i + 1) * n].view(qr, qw) for i in range(3)))
        off += 3 * n
    qw, qr = w >> levels, rows >> levels
    return out, slice_[off: off + qw * qr].view(qr, qw)


def stitch_strip_pyramid(slices, w, h, levels):
    """Concatenates the ranks' slices (rank order) into the flat
    multi_level_forward layout (Pyramid.flat)."""
    import torch
    n = len(slices)
    rows = h // n
    parts = [strip_slice_planes(s, w, rows, levels) for s in slices]
    flat = []
    for l in range(levels):
        for i in range(3):
            flat.append(torch.cat([p[0][l][i] for p in parts], 0).reshape(-1))
    flat.append(torch.cat([p[1] for p in parts], 0).reshape(-1))
    return torch.cat(flat)


def strip_pyramid_distributed(img_rows, w, h, levels, scheme: Scheme, group=None,
                              apply_scaling=False, boundary="periodic"):
    """Builds and connects this rank's StripPyramid over torch.distributed
    (blobs exchanged with all_gather_object; ring neighbours) and fills its
    input with `img_rows` (rows x w on this rank's GPU)."""
    import torch.distributed as dist
    rank, n = dist.get_rank(group), dist.get_world_size(group)
    sp = StripPyramid(w, h, levels, scheme, rank, n, apply_scaling, boundary)
    if n > 1:
        blobs = [None] * n
        dist.all_gather_object(blobs, sp.export(), group=group)
        sp.connect(blobs[(rank - 1) % n], blobs[(rank + 1) % n])
    if img_rows is not None:
        sp.input.copy_(img_rows)
    return sp


# ------------------------------------------------------------ host buffers
def _host_f32(t, what):
    import torch
    if not isinstance(t, torch.Tensor) or t.is_cuda or t.dtype != torch.float32:
        raise ValueError(f"{what} must be a float32 CPU tensor")
    return t.contiguous()


def forward_host(img, scheme: Scheme, boundary="periodic", apply_scaling=False, out=None):
    """`forward` with HOST buffers (the reference's own call shape,
    transform.hpp:65-66): (h, w) float32 CPU tensor -> (4, h/2, w/2) CPU
    planes. Copies and kernels are pipelined in row chunks on the current
    device; pass pinned tensors (`pin_memory()`) for full PCIe overlap."""
    import torch
    img = _host_f32(img, "img")
    if img.dim() != 2:
        raise ValueError("img must be 2-D (height, width)")
    h, w = img.shape
    if out is None:
        out = torch.empty((4, max(h // 2, 0), max(w // 2, 0)), dtype=torch.float32)
    _check(lib().wl_dwt2_forward_host(
        img.data_ptr(), w, h, w, scheme.wavelet.index, scheme.kind,
        _index(BOUNDARIES, boundary, "boundary"), int(bool(apply_scaling)),
        out[0].data_ptr(), out[1].data_ptr(), out[2].data_ptr(), out[3].data_ptr(),
        out.stride(1)))
    return out


def inverse_host(q, wavelet, boundary="periodic", undo_scaling=False, scheme=None, out=None):
    """`inverse` with HOST buffers: (4, qh, qw) CPU planes -> (2qh, 2qw)."""
    import torch
    q = _host_f32(q, "q")
    if q.dim() != 3 or q.shape[0] != 4:
        raise ValueError("q must be (4, qh, qw)")
    w = wavelet if isinstance(wavelet, WaveletSpec) else get_wavelet(wavelet)
    _, qh, qw = q.shape
    if out is None:
        out = torch.empty((2 * qh, 2 * qw), dtype=torch.float32)
    _check(lib().wl_dwt2_inverse_host(
        q[0].data_ptr(), q[1].data_ptr(), q[2].data_ptr(), q[3].data_ptr(), qw, qh, qw, w.index,
        _kind(scheme), _index(BOUNDARIES, boundary, "boundary"), int(bool(undo_scaling)),
        out.data_ptr(), out.stride(0)))
    return out
