"""In-tree build of libwavelift_b200.so (sm_100a) and the CPU oracle.

`python -m paper_1605_00561_b200._build` or `__graft_entry__.build()`.
nvcc cross-compiles for sm_100a without a GPU; the .so lands next to this
file so it travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# WL_VARIANT=<tag> with WL_DEFS="-DX=1 ..." builds an A/B variant library
# (libwavelift_b200_<tag>.so) for tuning experiments; loaded via WL_LIB.
VARIANT = os.environ.get("WL_VARIANT", "")
# variant objects live OUTSIDE the repo (they must not travel to the GPU box)
OBJ = (os.path.join(os.environ.get("WL_OBJV", "/tmp/wl_objv"), VARIANT) if VARIANT
       else os.path.join(PKG, "_obj"))
LIB = os.path.join(PKG, "libwavelift_b200" + ("_" + VARIANT if VARIANT else "") + ".so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
                "--expt-relaxed-constexpr", "-Xptxas", "-v", "-ccbin", "g++",
                "-I" + os.path.join(ROOT, "include")] + os.environ.get("WL_DEFS", "").split()
SOURCES = ["wl_capi.cu", "wl_interp.cu", "wl_fast.cu", "wl_fast_cdf53_fwd.cu",
           "wl_fast_cdf53_inv.cu", "wl_fast_cdf97_fwd.cu", "wl_fast_cdf97_inv.cu", "wl_conv.cu", "wl_strips.cu", "wl_host.cu", "wl_desc.cu",
           "wl_fast_cdf53_direct.cu", "wl_fast_cdf97_direct.cu", "wl_fast_dd137_fwd.cu",
           "wl_fast_dd137_inv.cu", "wl_fast_dd137_direct.cu"]


def _deps():
    files = []
    for d in (CSRC, os.path.join(CSRC, "gen"), os.path.join(ROOT, "include")):
        if os.path.isdir(d):
            files += [os.path.join(d, f) for f in os.listdir(d)
                      if f.endswith((".h", ".cuh", ".hpp"))]
    return files


def _newer(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _compile(src, verbose):
    obj = os.path.join(OBJ, os.path.basename(src).replace(".cu", ".o"))
    if not _newer(obj, [src, *_deps(), __file__]):
        return obj, ""
    cmd = [NVCC, *FLAGS, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    log = r.stdout + r.stderr
    with open(obj + ".ptxas.txt", "w") as f:
        f.write(log)
    return obj, log if verbose else ""


def gen_tables():
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "gen_steps.py")], check=True,
                   capture_output=True)


def build_lib(verbose=False) -> str:
    gen_tables()
    os.makedirs(OBJ, exist_ok=True)
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    with ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        res = list(ex.map(lambda s: _compile(s, verbose), srcs))
    objs = [o for o, _ in res]
    for _, log in res:
        if log:
            print(log)
    if _newer(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-ccbin", "g++"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


CLI_SRC = os.path.join(PKG, "cli", "wavelift_b200.cpp")
CLI_BIN = os.path.join(PKG, "bin", "wavelift_b200")


def build_cli() -> str:
    """The wavelift_b200 CLI (host C++ over the C-ABI library)."""
    deps = [CLI_SRC, LIB, os.path.join(ROOT, "include", "wavelift_b200.hpp"),
            os.path.join(ROOT, "include", "wavelift_b200_io.hpp")]
    if not _newer(CLI_BIN, deps):
        return CLI_BIN
    os.makedirs(os.path.dirname(CLI_BIN), exist_ok=True)
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", "-o", CLI_BIN, CLI_SRC,
           "-I" + os.path.join(ROOT, "include"), "-I/usr/local/cuda/include", "-L" + PKG,
           "-lwavelift_b200", "-L/usr/local/cuda/lib64", "-lcudart",
           "-Wl,-rpath,$ORIGIN/..:/usr/local/cuda/lib64"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"CLI build failed:\n{r.stdout}\n{r.stderr}")
    return CLI_BIN


def build_oracle():
    r = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], capture_output=True,
                       text=True)
    if r.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{r.stdout}\n{r.stderr}")


def build(verbose=False):
    build_oracle()
    lib = build_lib(verbose)
    if not VARIANT:
        build_cli()
    return lib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
