#!/usr/bin/env python3
"""Generates tests/golden/* from the UNMODIFIED reference (oracle/_ref).

Run here (where /root/reference exists and `make -C oracle` built
oracle/_ref/libwavelift_ref.so); the outputs are committed so the CPU and GPU
test suites never need /root/reference at run time.

* schemes_ref.json -- build_scheme() of every wavelet x scheme
  (schemes.cpp:146-174): labels, barrier flags, 4x4 entries with exact and
  double coefficients, cost counts (count_barriers/count_macs), zeta, and the
  2-D convolution filters (wavelets.cpp:80-88).
* fwd_*.npz / inv_*.npz / pyr_*.npz -- reference outputs on the reference
  tests' own seeded inputs (proj/tests/test_util.hpp:58-74 generators,
  seeds from test_transform.cpp / acceptance.cpp).
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.oracle import BOUNDARIES, SCHEMES, WAVELETS, RefLib  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def main():
    ref = RefLib()
    os.makedirs(OUT, exist_ok=True)
    tables = {w: {s: ref.dump_scheme(w, s) for s in SCHEMES} for w in WAVELETS}
    with open(os.path.join(OUT, "schemes_ref.json"), "w") as f:
        json.dump(tables, f, indent=0, sort_keys=True)

    # Forward, every scheme x {cdf53, cdf97} x boundary, on the reference
    # tests' dyadic (seed 101, test_transform.cpp:131) and uniform (seed 102,
    # test_transform.cpp:145) 32x32 images.
    for tag, seed, dyadic in (("dyadic32", 101, True), ("random32", 102, False)):
        img = ref.random_image(32, 32, seed, dyadic)
        arrs = {"img": img}
        for w in ("cdf53", "cdf97"):
            for s in SCHEMES:
                for b in BOUNDARIES:
                    arrs[f"{w}/{s}/{b}"] = ref.forward(img, w, s, b, False)
        np.savez_compressed(os.path.join(OUT, f"fwd_{tag}.npz"), **arrs)

    # Scaling (test_transform.cpp:211-225, seed 107).
    img = ref.random_image(16, 16, 107, False)
    arrs = {"img": img}
    for w in ("cdf53", "cdf97"):
        for b in BOUNDARIES:
            arrs[f"{w}/sweldens/{b}"] = ref.forward(img, w, "sweldens", b, True)
    np.savez_compressed(os.path.join(OUT, "fwd_scaled16.npz"), **arrs)

    # Inverse on arbitrary planes (not a forward output), seed 109.
    planes = ref.random_image(16, 64, 109, False).reshape(4, 16, 16)
    arrs = {"planes": planes}
    for w in ("cdf53", "cdf97"):
        for b in BOUNDARIES:
            for undo in (0, 1):
                arrs[f"{w}/{b}/{undo}"] = ref.inverse(planes, w, b, bool(undo))
    np.savez_compressed(os.path.join(OUT, "inv_random16.npz"), **arrs)

    # Pyramids: 3-level cdf53 sweldens periodic on dyadic 64x32 seed 110
    # (test_transform.cpp:273-305) and cdf97 monolithic_star symmetric.
    img = ref.random_image(64, 32, 110, True)
    arrs = {"img": img}
    for w, s, b in (("cdf53", "sweldens", "periodic"), ("cdf53", "monolithic", "symmetric"),
                    ("cdf97", "monolithic_star", "periodic"),
                    ("cdf97", "monolithic_star", "symmetric")):
        flat = ref.pyramid_forward(img, w, s, 3, b, False)
        arrs[f"fwd/{w}/{s}/{b}"] = flat
        arrs[f"inv/{w}/{s}/{b}"] = ref.pyramid_inverse(flat, 64, 32, 3, w, b, False)
    np.savez_compressed(os.path.join(OUT, "pyr_dyadic64x32.npz"), **arrs)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
