"""Barrier structure on real SASS (the reference checks it on its simulator,
acceptance.cpp:236-254 / test_parsim.cpp:101-115): every fast-engine kernel
contains exactly count_barriers(scheme) block barriers: per tile, the
data-availability barrier is an mbarrier phase wait on the TMA stage
(SYNCS.PHASECHK, counted separately) and every epoch after the first is one
named bar.sync of the compute warps (count_barriers - 1 of them); the one
CTA-wide bar.sync after the mbarrier initialisation completes the total. The
compile-time negative control WL_BREAK_BARRIER drops exactly one (racecheck
flags the resulting hazard: test_gpu_race.py). CPU-only: cuobjdump on the
built library."""
import os
import re
import shutil
import subprocess

import pytest

import paper_1605_00561_b200 as wl

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUOBJDUMP = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"


def barrier_counts(lib_path):
    """{(wavelet, scheme, dir, mangled name): BAR count} for every fast
    kernel -- each program has a plain, a symmetric-border (mirroring) and a
    direct-load instantiation, checked separately."""
    out = subprocess.run([CUOBJDUMP, "-sass", lib_path], capture_output=True, text=True,
                         check=True).stdout
    counts, fn = {}, None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            name = m.group(1)
            km = re.search(r"fast_kernelI\d+P_(cdf\d+|dd137)_(\w+?)_(fwd|inv)", name)
            fn = km.groups() + (name,) if km else None
            if fn:
                counts.setdefault(fn, 0)
                kinds_of.setdefault(fn, {"init": 0, "epoch": 0, "wait": 0})
            continue
        if fn and re.search(r"\bBAR\.(SYNC|RED|ARV)", line):
            counts[fn] += 1
            # bar.sync 0: the one CTA-wide barrier after the mbarrier init;
            # bar.sync 1, NW*32: the per-tile epoch barriers of the compute warps
            kinds_of[fn]["init" if re.search(r"BAR\.SYNC\S* 0x0 ;", line) else "epoch"] += 1
        if fn and re.search(r"SYNCS\.PHASECHK", line):
            kinds_of[fn]["wait"] += 1  # mbarrier waits (the per-tile data availability)
    return counts


kinds_of = {}  # (wavelet, scheme, dir, name) -> {"init", "epoch", "wait"} (barrier_counts)


@pytest.mark.skipif(not os.path.exists(CUOBJDUMP), reason="cuobjdump not available")
def test_sass_barriers_equal_count_barriers():
    counts = barrier_counts(wl.LIB_PATH)
    programs = {k[:3] for k in counts}
    # cdf53 / cdf97: 9 lifting schemes x 2 directions; dd137: 7 (Polyphase(*)
    # stays on the interpreter)
    assert len(programs) == 2 * 9 * 2 + 7 * 2, sorted(programs)
    # cdf53 / cdf97: plain + mirroring + direct-load variant; dd137 (reach 2):
    # plain + direct-load
    assert len(counts) == 3 * 36 + 2 * 14, len(counts)
    kinds = {"direct": 0, "mirror": 0}
    for (w, s, d, name), n in counts.items():
        want = wl.build_scheme(s, w).info(0 if d == "fwd" else 1)["barriers"]
        xf, mirror, direct = variant_flags(name)
        kinds["direct"] += direct
        kinds["mirror"] += mirror
        assert n == want, (w, s, d, n, want)
        # per tile: the data-availability wait (an mbarrier phase wait, not a
        # bar.sync; the direct-load variant loads its own cells) + one named
        # barrier per epoch after the first; plus the single init barrier
        k = kinds_of[(w, s, d, name)]
        assert k["init"] == 1 and k["epoch"] == want - 1, (w, s, d, k, want)
        assert direct or k["wait"] >= 1, (w, s, d, k)
    assert kinds == {"direct": 36 + 14, "mirror": 36}, kinds


def variant_flags(name):
    """(XF, MIRROR, DIRECT) template flags of a mangled fast_kernel."""
    m = re.search(r"Lb(\d)ELb(\d)ELb(\d)EEEv14CUtensorMap", name)
    assert m, name
    return tuple(int(x) for x in m.groups())


def build_broken(epoch=1):
    env = dict(os.environ, WL_VARIANT=f"brk{epoch}", WL_DEFS=f"-DWL_BREAK_BARRIER={epoch}")
    subprocess.run([os.sys.executable, "-m", "paper_1605_00561_b200._build"], cwd=ROOT, env=env,
                   check=True, capture_output=True)
    return os.path.join(ROOT, "paper_1605_00561_b200", f"libwavelift_b200_brk{epoch}.so")


@pytest.mark.skipif(not os.path.exists(CUOBJDUMP), reason="cuobjdump not available")
def test_broken_barrier_variant_drops_one_barrier():
    lib = build_broken(1)
    counts = barrier_counts(lib)
    for (w, s, d, name), n in counts.items():
        want = wl.build_scheme(s, w).info(0 if d == "fwd" else 1)["barriers"]
        # epoch 1 exists only for schemes with >= 2 barriers
        want = want - 1 if want >= 2 else want
        assert n == want, (w, s, d, n, want)
