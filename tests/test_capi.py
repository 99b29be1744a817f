"""CPU-side checks of the C-ABI library: it loads, exports every symbol that
include/wl_dwt.h declares, and the host-only entry points (validation,
metadata) behave like the reference -- no compute is launched here."""
import ctypes
import os
import re

import pytest

import paper_1605_00561_b200 as wl
from paper_1605_00561_b200 import schemes as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "wl_dwt.h")).read()
    return sorted(set(re.findall(r"\b(wl_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = wl.lib()
    names = declared_symbols()
    assert len(names) >= 12
    for n in names:
        assert hasattr(lib, n), n


def test_version_and_engine():
    assert "sm_100a" in wl.version()
    prev = wl.set_engine(1)
    assert wl.set_engine(prev) == 1


def test_resolve_index_matches_reference_table():
    # proj/tests/test_transform.cpp:28-51
    assert [wl.resolve_index(i, 4, "symmetric") for i in (-5, -2, -1, 0, 4, 5, 6, 7)] == \
        [1, 2, 1, 0, 2, 1, 0, 1]
    assert [wl.resolve_index(i, 4, "periodic") for i in (-5, -1, 4, 9)] == [3, 3, 0, 1]
    assert wl.resolve_index(-3, 1, "symmetric") == 0


def test_scheme_info_matches_reference_cost_table():
    # acceptance.cpp:62-67 (frozen) -- barriers and MACs of every cell
    want = {"cdf53": [(4, 16), (3, 24), (3, 18), (3, 24), (3, 18), (2, 24), (2, 18), (1, 63),
                      (1, 23), (1, 64)],
            "cdf97": [(8, 32), (6, 48), (6, 36), (6, 48), (6, 36), (4, 48), (4, 36), (2, 126),
                      (2, 46), (1, 256)],
            "dd137": [(4, 32), (3, 64), (3, 50), (3, 64), (3, 50), (2, 64), (2, 50), (1, 255),
                      (1, 203), (1, 256)]}
    for w, rows in want.items():
        for s, (b, m) in zip(S.SCHEMES, rows):
            info = wl.build_scheme(s, w).info()
            assert (info["barriers"], info["macs"]) == (b, m), (w, s)
            # one block barrier per neighbour-reading step: epochs == barriers
            assert info["epochs"] == b, (w, s)
            inv = wl.build_scheme(s, w).info(direction=1)
            assert inv["epochs"] == (b if s != "convolution" else want[w][0][0]), (w, s)


def test_halo_matches_required_halo():
    # parsim required_halo: 1 / 2 / 3 for cdf53 / cdf97 / dd137 (test_parsim.cpp:230-240)
    for w, h in (("cdf53", 1), ("cdf97", 2), ("dd137", 3)):
        for s in S.SCHEMES[:9]:
            assert wl.build_scheme(s, w).info()["halo"] == h


def test_validation_errors_without_gpu():
    lib = wl.lib()
    fp = ctypes.c_void_p(1)  # never dereferenced: validation fails first
    st = lib.wl_dwt2_forward(fp, 5, 4, 5, 0, 0, 0, 0, fp, fp, fp, fp, 2, None)
    assert st == wl.WL_EINVAL and b"even positive" in lib.wl_last_error()
    st = lib.wl_dwt2_forward(fp, 4, 4, 4, 7, 0, 0, 0, fp, fp, fp, fp, 2, None)
    assert st == wl.WL_EINVAL
    st = lib.wl_dwt2_pyramid_forward(fp, 12, 16, 3, 0, 0, 0, 0, fp, fp, None)
    assert st == wl.WL_EINVAL and b"2^levels" in lib.wl_last_error()
    st = lib.wl_dwt2_pyramid_forward(fp, 16, 16, 0, 0, 0, 0, 0, fp, fp, None)
    assert st == wl.WL_EINVAL and b"levels" in lib.wl_last_error()
    assert lib.wl_pyramid_elems(64, 32, 3) == 64 * 32


def test_selection_surface():
    assert wl.scheme_name(6) == "monolithic_star"
    assert wl.parse_scheme("polyphase_star") == 8 and wl.parse_scheme("nope") is None
    assert wl.parse_boundary("symmetric") == 1 and wl.boundary_name(0) == "periodic"
    with pytest.raises(ValueError):
        wl.get_wavelet("haar")
    assert abs(wl.get_wavelet("cdf97").zeta - 1.149604398860241) < 1e-15


def test_new_entry_points_validate_without_gpu():
    """Batch / strip / host / strips-runtime entry points reject bad arguments
    with WL_EINVAL before touching the device (reference error classes)."""
    lib = wl.lib()
    fp = ctypes.c_void_p(1)  # never dereferenced
    st = lib.wl_dwt2_forward_batch(fp, 8, 8, 8, 64, -1, 0, 0, 0, 0, fp, fp, fp, fp, 4, 16, None)
    assert st == wl.WL_EINVAL and b"batch" in lib.wl_last_error()
    st = lib.wl_dwt2_forward_batch(fp, 8, 8, 8, 32, 2, 0, 0, 0, 0, fp, fp, fp, fp, 4, 16, None)
    assert st == wl.WL_EINVAL and b"stride" in lib.wl_last_error()     # img stride < pitch*h
    assert lib.wl_dwt2_forward_batch(fp, 8, 8, 8, 64, 0, 0, 0, 0, 0, fp, fp, fp, fp, 4, 16,
                                     None) == wl.WL_OK                   # empty batch: no-op
    st = lib.wl_dwt2_pyramid_forward_batch(fp, 24, 12, 288, 2, 3, 0, 0, 0, 0, fp, 288, fp, None)
    assert st == wl.WL_EINVAL and b"2^levels" in lib.wl_last_error()
    st = lib.wl_dwt2_forward_strip(fp, 64, 32, 2, 64, 1, 6, 0, fp, fp, fp, fp, 32, None)
    assert st == wl.WL_EINVAL and b"halo" in lib.wl_last_error()       # cdf97 needs 6 rows
    st = lib.wl_dwt2_forward_strip(fp, 64, 31, 6, 64, 1, 6, 0, fp, fp, fp, fp, 32, None)
    assert st == wl.WL_EINVAL                                          # odd rows
    st = lib.wl_dwt2_inverse_strip(fp, fp, fp, fp, 32, 16, 1, 32, 1, 6, 0, fp, 64, None)
    assert st == wl.WL_EINVAL                                          # cdf97 inverse needs 3
    st = lib.wl_dwt2_forward_host(fp, 7, 8, 7, 0, 0, 0, 0, fp, fp, fp, fp, 4)
    assert st == wl.WL_EINVAL and b"even" in lib.wl_last_error()
    st = lib.wl_dwt2_inverse_host(None, fp, fp, fp, 4, 4, 4, 0, 0, 0, 0, fp, 8)
    assert st == wl.WL_EINVAL and b"null" in lib.wl_last_error()
    # ping-pong LL planes: level-1-size and level-2-size planes per image
    assert lib.wl_pyramid_batch_scratch_elems(64, 64, 2, 3) == 3 * (32 * 32 + 16 * 16)
    assert lib.wl_pyramid_batch_scratch_elems(64, 64, 1, 3) == 3 * 32 * 32
