"""File formats and the wavelift_b200 CLI.

CPU: the PGM / subband-container code of the drop-in writes byte-identical
files to the unmodified reference and reads the reference's files
(tests/cpp/test_io.cpp); the CLI builds and rejects bad arguments with the
reference's exit codes. GPU: `wavelift_b200 transform` writes the same file
as the reference's cmd_transform (header byte-identical, payload bit-exact
for cdf53 on an 8-bit image, within tolerance for cdf97), and the
sweldens/monolithic payloads are byte-identical (cli_smoke.sh:108-120)."""
import ctypes
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref", "libwavelift_ref.so")
CLI = os.path.join(ROOT, "paper_1605_00561_b200", "bin", "wavelift_b200")
need_ref = pytest.mark.skipif(not os.path.exists(REF), reason="oracle/_ref not built")


def write_pgm(path, px, maxval=255):
    h, w = px.shape
    with open(path, "wb") as f:
        f.write(f"P5\n{w} {h}\n{maxval}\n".encode())
        f.write(px.astype(">u2" if maxval > 255 else "u1").tobytes())


@need_ref
def test_io_formats_match_reference(tmp_path):
    exe = str(tmp_path / "test_io")
    subprocess.run(["g++", "-std=c++17", "-O1", "-o", exe,
                    os.path.join(ROOT, "tests", "cpp", "test_io.cpp"),
                    "-I" + os.path.join(ROOT, "include"), "-I/usr/local/cuda/include",
                    "-L" + os.path.dirname(REF), "-lwavelift_ref", "-L/usr/local/cuda/lib64",
                    "-lcudart", f"-Wl,-rpath,{os.path.dirname(REF)}:/usr/local/cuda/lib64"],
                   check=True, capture_output=True, text=True)
    r = subprocess.run([exe, str(tmp_path)], capture_output=True, text=True)
    assert r.returncode == 0 and "PASS" in r.stdout, r.stdout + r.stderr


def run_cli(*args):
    return subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=600)


def test_cli_usage_errors(tmp_path):
    if not os.path.exists(CLI):
        pytest.skip("CLI not built")
    assert run_cli().returncode == 1
    assert run_cli("nope").returncode == 1
    odd = tmp_path / "odd.pgm"
    write_pgm(odd, np.zeros((5, 6), np.uint16))
    r = run_cli("transform", odd, tmp_path / "o.sub")
    assert r.returncode == 1 and "--pad" in r.stderr          # invalid_argument -> 1
    r = run_cli("transform", odd, tmp_path / "o.sub", "--scheme", "bogus")
    assert r.returncode == 1 and "unknown scheme" in r.stderr
    r = run_cli("transform", tmp_path / "missing.pgm", tmp_path / "o.sub")
    assert r.returncode == 2                                   # runtime_error -> 2


def read_sub(path):
    data = open(path, "rb").read()
    head, payload = data.split(b"data\n", 1)
    return head, np.frombuffer(payload, "<f8")


@pytest.mark.gpu
@need_ref
def test_cli_transform_matches_reference_cmd_transform(tmp_path):
    ref = ctypes.CDLL(REF)
    rng = np.random.default_rng(3)
    img = rng.integers(0, 256, size=(64, 96)).astype(np.uint16)
    pgm = tmp_path / "in.pgm"
    write_pgm(pgm, img)
    for wavelet, wid, levels, exact in (("cdf53", 0, 2, True), ("cdf97", 1, 3, False)):
        for scheme, sid in (("sweldens", 0), ("monolithic", 5), ("monolithic_star", 6)):
            for boundary, bid in (("periodic", 0), ("symmetric", 1)):
                ours, theirs = tmp_path / "ours.sub", tmp_path / "ref.sub"
                r = run_cli("transform", pgm, ours, "--wavelet", wavelet, "--scheme", scheme,
                            "--levels", levels, "--boundary", boundary)
                assert r.returncode == 0 and "wrote" in r.stdout, r.stderr
                assert ref.wlref_transform_file(str(pgm).encode(), str(theirs).encode(), wid, sid,
                                                levels, bid, 0) == 0
                h1, p1 = read_sub(ours)
                h2, p2 = read_sub(theirs)
                assert h1 == h2
                if exact:
                    assert np.array_equal(p1, p2), (scheme, boundary)
                else:
                    assert np.abs(p1 - p2).max() <= 1e-5 * (p2.max() - p2.min())
    # cli_smoke.sh:108-120: sweldens and monolithic payloads byte-identical
    small = tmp_path / "s.pgm"
    write_pgm(small, rng.integers(0, 256, size=(16, 16)).astype(np.uint16))
    run_cli("transform", small, tmp_path / "a.sub", "--scheme", "sweldens")
    run_cli("transform", small, tmp_path / "b.sub", "--scheme", "monolithic")
    assert read_sub(tmp_path / "a.sub")[1].tobytes() == read_sub(tmp_path / "b.sub")[1].tobytes()


@pytest.mark.gpu
def test_cli_roundtrip_and_bench(tmp_path):
    rng = np.random.default_rng(4)
    pgm = tmp_path / "in.pgm"
    write_pgm(pgm, rng.integers(0, 4096, size=(128, 64)).astype(np.uint16), maxval=4095)
    for w in ("cdf53", "cdf97"):
        r = run_cli("roundtrip", pgm, "--wavelet", w, "--scheme", "monolithic_star", "--levels", 3)
        assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr
    # wavelift_main.cpp:196: the reference inverts with the wavelet-only
    # (Sweldens) inverse, so a symmetric Polyphase roundtrip FAILs (exit 2)
    # there (the oracle: max error 0.12); --scheme-inverse runs the scheme's
    # own inverse kernel instead.
    r = run_cli("roundtrip", pgm, "--scheme", "polyphase", "--boundary", "symmetric")
    assert r.returncode == 2 and "FAIL" in r.stdout and "note:" in r.stderr, r.stdout
    r = run_cli("roundtrip", pgm, "--scheme", "monolithic", "--boundary", "symmetric",
                "--scheme-inverse")
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr
    r = run_cli("bench", "--size", "2048x1024", "--wavelet", "cdf97", "--scheme",
                "monolithic_star", "--reps", 3, "--format", "csv")
    lines = r.stdout.splitlines()
    assert r.returncode == 0 and lines[0] == "scheme,wavelet,size,mbps", r.stderr
    assert lines[1].startswith("monolithic_star,cdf97,2048x1024,") and lines[1].count(",") == 3
    r = run_cli("bench", "--size", "256x256", "--reps", 2)
    assert r.returncode == 0 and r.stdout.rstrip().endswith("over 2 rep(s)"), r.stdout
    r = run_cli("bench", "--size", "256x256", "--reps", 2, "--format", "csv", "--gpix")
    assert r.stdout.splitlines()[0] == "scheme,wavelet,size,mbps,gpix_s", r.stdout
