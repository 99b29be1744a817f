#!/usr/bin/env python3
"""Benchmark of the B200 2-D lifting DWT (BASELINE.json metric/configs).

Workload (N=1, BASELINE.json configs[1]): one STEP = every scheme x {cdf53,
cdf97} (20 programs), each a single-level forward then that scheme's inverse
of a 8192x8192 float32 image (periodic boundary, scaling off, as the
reference's cmd_bench, wavelift_main.cpp:236-272). 40 passes of 67.1 MPix.

* value      GPixel/s = input pixels of all passes / device time of the step
             (inputs resident in HBM; inputs > L2, so no flush needed).
* e2e        same metric through the public API with HOST (pinned) buffers:
             each pass copies its input H2D and its result D2H inside the
             timed region; pcie = the box's plain pinned-copy ceiling.
* per_scheme [ms, GPix/s, fraction of the HBM copy peak] per program, each
             program timed ISOLATED: back-to-back launches of that program
             alone (warm), median of the CUDA-event launch times.
* roofline   dominant kernel of the step (largest share of step time):
             algorithmic bytes = 8 B/pixel (one f32 read + one f32 write per
             pixel) / its isolated median launch time, against
             the measured HBM copy peak (MEASURED_PEAKS.json).
* cpu_baseline  the unmodified reference (oracle/_ref, "reference") on the
             host cores at the FULL configs[1] size for the headline pair
             (cdf53 Monolithic, cdf97 Monolithic*; forward + reference
             inverse), with the GPU's isolated times of the same programs.
* north_star (last key, so it survives a tail-truncated log)
             c3 = configs[2] (16384^2: cdf97 Monolithic*, Monolithic,
             Sweldens; cdf53 Monolithic, Monolithic*; fwd & inv, each with
             its fraction of the copy peak and ncu DRAM traffic ratio),
             c4 = configs[3] (32768^2 5-level strip pyramid),
             c5 = configs[4] (4096 x 4096^2 3-level batches).

`--impl reference` times the reference's CPU implementation of the SAME step
(same config object) on a bounded sample: every program forward + reference
inverse on an 8192-wide band of --ref-rows rows per step (rank 0 only under
torchrun).
Multi-GPU (torchrun): every rank runs the full step on its own image(s)
(independent images, no data-path collective; weak scaling); time = max over
ranks of the device time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "2-D DWT GPixel/s and ns/pixel per scheme; % of B200 HBM BW; 1/2/4/8 GPU"
WAVELETS = ("cdf53", "cdf97")
SCHEMES = ("sweldens", "iwahashi", "iwahashi_star", "explosive", "explosive_star",
           "monolithic", "monolithic_star", "polyphase", "polyphase_star", "convolution")
SIZE = 8192
C3 = 16384


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, index=0):
        self.samples, self.proc, self.index = [], None, index

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.samples and time.time() - t0 < 5:  # sampler is live
                time.sleep(0.01)
            self.samples.clear()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(s[0]) for s in self.samples if s and s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if len(s) > 1 and s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for n, v in zip(names, s[3:7]):
                if v.strip().lower() == "active":
                    reasons.add(n)
        # samples under load only (the GPU idles between nvidia-smi start and the loop)
        load = [x for x in sm if mx and x > 0.5 * max(mx)] or sm
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_init():
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # WL_BENCH_DEVICE / WL_BENCH_BACKEND: test hooks to run N ranks on one
    # GPU (gloo for the timing barrier; NCCL refuses duplicate devices).
    dev = int(os.environ.get("WL_BENCH_DEVICE", local))
    backend = os.environ.get("WL_BENCH_BACKEND", "nccl")
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(dev)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(dev)
    return ws, rank, dev


def barrier_max(x, ws):
    """max over ranks of a float (device-timed ms)."""
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    on_gpu = dist.get_backend() == "nccl"
    t = torch.tensor([x], device="cuda" if on_gpu else "cpu", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


# ------------------------------------------------------------ shared config
PROGRAMS = [(w, s) for w in WAVELETS for s in SCHEMES]
# the reference CPU timed at the full configs[1] size (the headline pair)
CPU_FULL = (("cdf53", "monolithic"), ("cdf97", "monolithic_star"))
# dd137 schemes on the fast engine (Polyphase(*) of reach 3 stay on the interpreter)
DD137_FAST = ("sweldens", "iwahashi", "iwahashi_star", "explosive", "explosive_star",
              "monolithic", "monolithic_star")
# configs[2] ablation at 16384^2: the north-star kernels and their neighbours
C3_PROGRAMS = (("cdf97", "monolithic_star"), ("cdf97", "monolithic"), ("cdf97", "sweldens"),
               ("cdf53", "monolithic"), ("cdf53", "monolithic_star"))


def workload_config(n, ws):
    """The step's config object -- identical in both arms (--impl b200 and
    --impl reference), which time the same workload."""
    return {"workload": f"configs[1]: every scheme x {{cdf53, cdf97}}, single-level forward + "
                        f"that scheme's inverse, {n}x{n} float32 per rank, periodic, no scaling",
            "size": n, "programs": len(PROGRAMS),
            "pixels_per_step_per_rank": 2 * len(PROGRAMS) * n * n,
            "l2": "inputs (256 MiB) larger than L2 (126 MB); no flush",
            "parallelism": f"independent images, {ws} rank(s)"}


def traffic_of(key):
    """ncu DRAM bytes (read + write) per launch for `key`, from the newest
    profiles/traffic_rNN.json (one `ncu --set full` capture per kernel)."""
    for r in ("r02", "r01"):
        path = os.path.join(ROOT, "profiles", f"traffic_{r}.json")
        if os.path.exists(path):
            try:
                v = json.load(open(path)).get(key)
            except Exception:
                v = None
            if v is not None:
                return v
    return None


# --------------------------------------------------------------- reference arm
def reference_step_sample(ref, img):
    """One bounded sample of the step on the reference CPU path: every scheme
    x wavelet forward (transform.cpp:163) then the reference inverse
    (transform.cpp:178, wavelet-only)."""
    px = 0
    for w in WAVELETS:
        for s in SCHEMES:
            q = ref.forward(img, w, s, "periodic", False)
            ref.inverse(q, w, "periodic", False)
            px += 2 * img.size
    return px


def _ref_lib():
    from oracle.oracle import Oracle, RefLib
    try:
        ref = RefLib()
        return ref, "reference", ref.worker_count()
    except FileNotFoundError:
        o = Oracle()
        return o, "port", int(o.lib.wlo_threads())


def run_reference(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import numpy as np
    n, rows = args.size, args.ref_rows
    ref, kind, cores = _ref_lib()
    # a band of the configs[1] image: full 8192-pixel rows, --ref-rows rows
    # (periodic), so every per-row cost is the full-size one; the whole
    # --steps/--warmup run stays within a few minutes
    img = np.random.default_rng(12345).random((rows, n))
    for _ in range(args.warmup):
        reference_step_sample(ref, img)
    times, px = [], 0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        px = reference_step_sample(ref, img)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    gpix = px * args.steps / tot / 1e9
    sample = (f"per step: a {n}x{rows} band (full {n}-pixel rows) of the {n}x{n} configs[1] "
              f"workload, float64 uniform[0,1) (numpy seed 12345); every scheme x {{cdf53,cdf97}} "
              f"forward + the reference inverse; periodic, no scaling; "
              f"WAVELIFT_THREADS={os.environ.get('WAVELIFT_THREADS', 'unset')} -> {cores} "
              f"worker threads")
    line = {"impl": "reference", "metric": METRIC, "value": gpix, "unit": "GPixel/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "ns_per_pixel": 1e9 * tot / (px * args.steps),
            "config": workload_config(n, ws),
            "cpu_baseline": {"value": gpix, "unit": "GPixel/s", "cores": cores, "kind": kind,
                             "sample": sample},
            "e2e": {"value": gpix, "unit": "GPixel/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------- GPU arm
# GPU sleep (~5 ms at 1.9 GHz) enqueued before a timed region: device time of
# back-to-back launches, without the host's first-launch latency.
PRIME_CYCLES = 10_000_000


def time_isolated(fn, stream, groups=5, per_group=10, warm=2):
    """Steady-state device time (ms) of one call of fn: `groups` groups of
    `per_group` back-to-back calls (no host sync in between), each group
    between two CUDA events on the launching stream; median of the group
    means (a single launch between two events is quantised to ~2 us)."""
    import torch
    for _ in range(warm):
        fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(groups)]
    for a, b in ev:
        # the group is enqueued while the GPU sleeps, so the host latency of
        # the first call is not inside the group (it is an e2e cost)
        torch.cuda._sleep(PRIME_CYCLES)
        a.record(stream)
        for _ in range(per_group):
            fn()
        b.record(stream)
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) / per_group for a, b in ev)


def prog_entry(t_ms, n, peak, traffic=None):
    gbs = 8.0 * n * n / (t_ms * 1e-3) / 1e9
    e = {"ms": round(t_ms, 5), "gpix_s": round(n * n / t_ms / 1e6, 1),
         "hbm_gbs": round(gbs, 1), "frac": round(gbs / peak, 4)}
    if traffic is not None:
        e["traffic_ratio"] = round(traffic / (8.0 * n * n), 3)
    return e


def run_gpu(args):
    import torch

    import paper_1605_00561_b200 as wl

    ws, rank, local = dist_init()
    peak, peak_src = peaks()
    dev = torch.device("cuda", local)
    n = args.size
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    img = torch.rand((n, n), device=dev, generator=g, dtype=torch.float32)
    rec = torch.empty_like(img)
    q = torch.empty((4, n // 2, n // 2), device=dev, dtype=torch.float32)
    schemes = {(w, s): wl.build_scheme(s, w) for (w, s) in PROGRAMS}
    stream = torch.cuda.current_stream()

    def step():
        for (w, s) in PROGRAMS:
            wl.forward(img, schemes[(w, s)], "periodic", False, out=q)
            wl.inverse(q, w, "periodic", False, scheme=s, out=rec)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    barrier(ws)

    # ---- timed region: K steps, device time, max over ranks
    n0 = wl.launch_count()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        barrier(ws)
        torch.cuda.synchronize()
        torch.cuda._sleep(PRIME_CYCLES)  # the host enqueues ahead of the GPU from the start
        start.record(stream)
        for _ in range(args.steps):
            step()
        stop.record(stream)
        torch.cuda.synchronize()
        barrier(ws)
    launches = wl.launch_count() - n0
    clocks = clk.summary()
    ms = start.elapsed_time(stop) / args.steps
    ms = barrier_max(ms, ws)
    px_step = 2 * len(PROGRAMS) * n * n
    value = ws * px_step / (ms * 1e-3) / 1e9

    # ---- per-program times: each program ISOLATED (back-to-back launches of
    # that program alone, warm), median of the CUDA-event launch times
    per, per_ms = {}, {}
    for (w, s) in PROGRAMS:
        sch = schemes[(w, s)]
        tf = time_isolated(lambda: wl.forward(img, sch, "periodic", False, out=q), stream)
        ti = time_isolated(lambda: wl.inverse(q, w, "periodic", False, scheme=s, out=rec),
                           stream)
        for d, t in (("fwd", tf), ("inv", ti)):
            key = f"{w}/{s}/{d}"
            per_ms[key] = t
            e = prog_entry(t, n, peak)
            per[key] = [e["ms"], e["gpix_s"], e["frac"]]

    # dominant kernel = largest share of the step, per actual kernel: the
    # Convolution scheme's inverse is the reference inverse (the Sweldens
    # inverse kernel), so both programs' launches count for that kernel
    def kernel_of(prog):
        w_, s_, d_ = prog.split("/")
        return f"{w_}/sweldens/inv" if (s_ == "convolution" and d_ == "inv") else prog
    share = {}
    for k, t in per_ms.items():
        share[kernel_of(k)] = share.get(kernel_of(k), 0.0) + t
    dom = max(share, key=share.get)
    dom_t = per_ms[dom]
    step_sum = sum(per_ms.values())
    dom_e = prog_entry(dom_t, n, peak)
    # FP32 side of the same kernel: MACs per quad (count_macs, schemes.cpp:176)
    # -> FMA per pixel = MACs / 4; FP32 peak = SMs x 128 FMA/clk x 2 x SM clock.
    dw, ds, dd = dom.split("/")
    macs = schemes[(dw, ds)].info(0 if dd == "fwd" or ds == "convolution" else 1)["macs"]
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    clk_hz = (clocks.get("sm_max_mhz") or 1965.0) * 1e6
    fp32_peak = sms * 128 * 2 * clk_hz / 1e12
    fp32 = 2.0 * macs / 4.0 * n * n / (dom_t * 1e-3) / 1e12
    roofline = {"bound": "hbm", "kernel": dom, "achieved": dom_e["hbm_gbs"], "peak": peak,
                "peak_source": peak_src, "unit": "GB/s", "frac": dom_e["frac"],
                "traffic": traffic_of(dom), "share_of_step": round(share[dom] / step_sum, 4),
                "launches_per_step": sum(1 for k in per_ms if kernel_of(k) == dom),
                "algorithmic_bytes_per_launch": 8.0 * n * n,
                "timing": "isolated steady state: median over 5 groups of 10 back-to-back launches "
                          "of this kernel alone (CUDA events around each group, each group "
                          "enqueued behind a GPU sleep so no host launch latency is inside)",
                "fp32": {"fma_per_px": macs / 4.0, "achieved_tflops": round(fp32, 2),
                         "peak_tflops": round(fp32_peak, 1), "sms": sms,
                         "frac": round(fp32 / fp32_peak, 4)}}

    # ---- C3: 16384^2 (configs[2]) -- the north-star kernels
    c3 = None
    if args.c3:
        big = torch.rand((C3, C3), device=dev, generator=g, dtype=torch.float32)
        qb = torch.empty((4, C3 // 2, C3 // 2), device=dev, dtype=torch.float32)
        rb = torch.empty_like(big)
        c3 = {}
        for (w, s) in C3_PROGRAMS:
            sch = wl.build_scheme(s, w)
            tf = time_isolated(lambda: wl.forward(big, sch, out=qb), stream)
            ti = time_isolated(lambda: wl.inverse(qb, w, scheme=s, out=rb), stream)
            for d, t in (("fwd", tf), ("inv", ti)):
                key = f"{w}/{s}/{d}"
                c3[key] = prog_entry(t, C3, peak, traffic_of(f"c3/{key}"))
        del big, qb, rb
        torch.cuda.empty_cache()

    # ---- unaligned shapes (w = 2 mod 4: odd plane widths, no TMA): the fast
    # engine's direct-load variant, and the generic interpreter for scale
    unaligned = None
    if args.unaligned and ws == 1:
        unaligned = {}
        for m in (8190, 8194):
            im = torch.rand((m, m), device=dev, generator=g, dtype=torch.float32)
            qm = torch.empty((4, m // 2, m // 2), device=dev, dtype=torch.float32)
            rm = torch.empty_like(im)
            for (w, s) in CPU_FULL:
                sch = wl.build_scheme(s, w)
                tf = time_isolated(lambda: wl.forward(im, sch, out=qm), stream)
                ti = time_isolated(lambda: wl.inverse(qm, w, scheme=s, out=rm), stream)
                unaligned[f"{m}/{w}/{s}/fwd"] = prog_entry(tf, m, peak)
                unaligned[f"{m}/{w}/{s}/inv"] = prog_entry(ti, m, peak)
            if m == 8190:
                prev = wl.set_engine(1)
                sch = wl.build_scheme("monolithic_star", "cdf97")
                t = time_isolated(lambda: wl.forward(im, sch, out=qm), stream, groups=3,
                                  per_group=3)
                wl.set_engine(prev)
                unaligned["8190/cdf97/monolithic_star/fwd/interpreter"] = prog_entry(t, m, peak)
            del im, qm, rm

    # ---- dd137: the fast engine's reach-2 kernels for every
    # lifting scheme but Polyphase(*) (interpreter), 8192^2, same image; the
    # generic interpreter on one scheme for scale
    dd = None
    if args.dd137 and ws == 1:
        dd = {}
        for s in DD137_FAST:
            sch = wl.build_scheme(s, "dd137")
            tf = time_isolated(lambda: wl.forward(img, sch, out=q), stream)
            ti = time_isolated(lambda: wl.inverse(q, "dd137", scheme=s, out=rec), stream)
            dd[f"dd137/{s}/fwd"] = prog_entry(tf, n, peak)
            dd[f"dd137/{s}/inv"] = prog_entry(ti, n, peak)
        prev = wl.set_engine(1)
        sch = wl.build_scheme("monolithic_star", "dd137")
        t = time_isolated(lambda: wl.forward(img, sch, out=q), stream, groups=3, per_group=3)
        wl.set_engine(prev)
        dd["dd137/monolithic_star/fwd/interpreter"] = prog_entry(t, n, peak)
        sch = wl.build_scheme("polyphase", "dd137")
        t = time_isolated(lambda: wl.forward(img, sch, out=q), stream, groups=3, per_group=3)
        dd["dd137/polyphase/fwd/interpreter"] = prog_entry(t, n, peak)

    # ---- e2e through the public API with pinned host buffers
    e2e = None
    if args.e2e_steps > 0:
        e2e = run_e2e(args, wl, ws, img, schemes, px_step)

    c4 = run_c4(args, wl, ws, rank, peak) if args.c4 else None
    c5 = run_c5(args, wl, ws, rank, peak) if args.c5 else None

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        # configs[0]: 1024^2 cdf53 Sweldens forward on the GPU, isolated
        im0 = torch.rand((1024, 1024), device=dev, generator=g, dtype=torch.float32)
        q0 = torch.empty((4, 512, 512), device=dev, dtype=torch.float32)
        s0 = wl.build_scheme("sweldens", "cdf53")
        c0_ms = time_isolated(lambda: wl.forward(im0, s0, out=q0), stream)
        cpu = cpu_baseline(args, per_ms, c0_ms)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "GPixel/s", "n_gpus": ws,
                "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f32", "data": "synthetic",
                "ns_per_pixel": ms * 1e6 / px_step,
                "config": workload_config(n, ws),
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches, "gpu_launches_per_step": launches / args.steps,
                "clocks": clocks, "c4": c4, "c5": c5, "unaligned": unaligned, "dd137": dd,
                "per_scheme_unit": "[ms, GPix/s, frac of copy peak] per launch, isolated steady "
                                   "state (median of 5 groups of 10 back-to-back launches)",
                "per_scheme": per,
                "north_star": north_star(c3, c4, c5, unaligned, dd)}
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def north_star(c3, c4, c5, unaligned=None, dd=None):
    """Compact configs[2..4] summary, emitted LAST in the line."""
    out = {}
    if dd:
        out["dd137_unit"] = "8192^2: [ms, frac of copy peak]"
        out["dd137"] = {k: [v["ms"], v["frac"]] for k, v in dd.items()}
    if unaligned:
        out["unaligned_unit"] = "[ms, frac of copy peak] (8190^2 / 8194^2 images: no TMA)"
        out["unaligned"] = {k: [v["ms"], v["frac"]] for k, v in unaligned.items()}
    if c3:
        out["c3_unit"] = "16384^2: [ms, frac of copy peak, ncu DRAM bytes / algorithmic]"
        out["c3"] = {k: [v["ms"], v["frac"], v.get("traffic_ratio")] for k, v in c3.items()}
    if c4:
        out["c4"] = {"ms": round(c4["ms"], 3), "gpix_s": round(c4["value"], 1),
                     "frac_per_gpu": round(c4["frac_per_gpu"], 4), "ranks": c4["ranks"]}
    if c5:
        out["c5"] = {w: {"ms": round(c5[w]["ms"], 2), "gpix_s": round(c5[w]["value"], 1),
                         "frac_per_gpu": round(c5[w]["frac_per_gpu"], 4)}
                     for w in ("cdf53", "cdf97") if w in c5}
    return out


def pcie_probe(nbytes):
    """The box's pinned-copy ceiling: H2D alone, D2H alone, both at once."""
    import torch
    h_a = torch.empty(nbytes // 4, dtype=torch.float32, pin_memory=True)
    h_b = torch.empty(nbytes // 4, dtype=torch.float32, pin_memory=True)
    d_a = torch.empty(nbytes // 4, device="cuda")
    d_b = torch.empty(nbytes // 4, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / 3

    def both():
        with torch.cuda.stream(s1):
            d_a.copy_(h_a, non_blocking=True)
        with torch.cuda.stream(s2):
            h_b.copy_(d_b, non_blocking=True)
    t_h2d = timed(lambda: d_a.copy_(h_a, non_blocking=True))
    t_d2h = timed(lambda: h_b.copy_(d_b, non_blocking=True))
    t_both = timed(both)
    return {"h2d_gbs": round(nbytes / t_h2d / 1e9, 1), "d2h_gbs": round(nbytes / t_d2h / 1e9, 1),
            "duplex_gbs_per_direction": round(nbytes / t_both / 1e9, 1), "bytes": nbytes}


def gpu_cpu_affinity(index):
    """Host CPUs local to GPU `index` (nvidia-smi topo -m "CPU Affinity"), or
    None. Pinned staging buffers touched from those CPUs land on the GPU's
    NUMA node."""
    try:
        out = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True,
                             timeout=10).stdout.splitlines()
        head = [h.strip() for h in out[0].split("\t")]
        col = next(i for i, h in enumerate(head) if h.startswith("CPU Affinity"))
        for line in out[1:]:
            f = [x.strip() for x in line.split("\t")]
            if f and f[0] == f"GPU{index}":
                cpus = set()
                for part in f[col].split(","):
                    a, _, b = part.partition("-")
                    cpus.update(range(int(a), int(b or a) + 1))
                return cpus & os.sched_getaffinity(0) or None
    except Exception:
        return None
    return None


def run_e2e(args, wl, ws, img, schemes, px_step):
    """The reference-facing call shape: forward(const Image&) /
    inverse(const QuadGrid&) on HOST buffers (wl_dwt2_forward_host /
    wl_dwt2_inverse_host: row-chunk pipeline, H2D/kernels/D2H overlap)."""
    import torch
    n = img.shape[0]
    # host side on the GPU's NUMA node (restored afterwards: the CPU
    # reference runs on every core)
    saved = os.sched_getaffinity(0)
    local = gpu_cpu_affinity(torch.cuda.current_device())
    if local:
        os.sched_setaffinity(0, local)
    try:
        return _run_e2e(args, wl, ws, img, schemes, px_step, n, local)
    finally:
        os.sched_setaffinity(0, saved)


def _run_e2e(args, wl, ws, img, schemes, px_step, n, local):
    import torch
    h_img = torch.empty((n, n), dtype=torch.float32, pin_memory=True)
    h_img.copy_(img.cpu())
    h_q = torch.empty((4, n // 2, n // 2), dtype=torch.float32, pin_memory=True)
    h_rec = torch.empty((n, n), dtype=torch.float32, pin_memory=True)

    def e2e_step():
        for (w, s) in PROGRAMS:
            wl.forward_host(h_img, schemes[(w, s)], out=h_q)    # host image -> host planes
            wl.inverse_host(h_q, w, scheme=s, out=h_rec)        # host planes -> host image

    e2e_step()
    torch.cuda.synchronize()
    barrier(ws)
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        e2e_step()  # synchronous calls: results are in host memory on return
    ems = barrier_max((time.perf_counter() - t0) * 1e3 / args.e2e_steps, ws)
    bytes_io = 2 * len(PROGRAMS) * 4 * n * n  # per direction per step
    pcie = pcie_probe(4 * n * n)
    gbs = bytes_io / (ems * 1e-3) / 1e9
    return {"value": ws * px_step / (ems * 1e-3) / 1e9, "unit": "GPixel/s",
            "ms_per_step": ems, "h2d_bytes_per_step": bytes_io, "d2h_bytes_per_step": bytes_io,
            "steps": args.e2e_steps, "h2d_gbs": round(gbs, 1), "d2h_gbs": round(gbs, 1),
            "pcie_ceiling": pcie,
            "frac_of_duplex_ceiling": round(gbs / pcie["duplex_gbs_per_direction"], 3),
            "host_cpus": (f"{len(local)} CPUs local to the GPU (nvidia-smi topo)" if local
                          else "all (GPU affinity unknown)"),
            "api": "forward_host / inverse_host (pinned host float32 buffers; wall clock "
                   "around synchronous calls); byte counts are the image/plane tensors, "
                   "the strip halo rows add <=1.2% H2D"}


def _timed(fn, steps, ws, stream):
    """device time (ms) per call of fn, max over ranks."""
    import torch
    barrier(ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return barrier_max(e0.elapsed_time(e1) / steps, ws)


def run_c4(args, wl, ws, rank, peak):
    """BASELINE configs[3]: cdf97 5-level pyramid of ONE N x N image split in
    row strips over the ranks, per-level halo exchange over peer memory
    (StripPyramid). Strong scaling: the image size is fixed."""
    import torch
    n, levels = args.c4_size, 5
    sch = wl.build_scheme("monolithic_star", "cdf97")
    if ws > 1:
        sp = wl.strip_pyramid_distributed(None, n, n, levels, sch)
    else:
        sp = wl.StripPyramid(n, n, levels, sch)
    # deterministic content by GLOBAL pixel coordinates: the same image for
    # every rank count, so the checksum is comparable across N
    rows = n // ws
    r_idx = torch.arange(rank * rows, (rank + 1) * rows, device="cuda", dtype=torch.int64)
    c_idx = torch.arange(n, device="cuda", dtype=torch.int64)
    h_ = (r_idx[:, None] * 1103515245 + c_idx[None, :] * 12345 + 2654435761) % 2147483647
    sp.input.copy_((h_ % 65536).float() / 65536.0)
    del h_
    out = torch.empty(sp.slice_elems(), device="cuda")
    stream = torch.cuda.current_stream()
    torch.cuda.synchronize()
    barrier(ws)  # every rank connected and idle before the first halo wait
    for _ in range(3):
        sp.forward(out)
    torch.cuda.synchronize()
    ms = _timed(lambda: sp.forward(out), max(args.steps, 5), ws, stream)
    sp.check()
    checksum = out.double().sum()
    if ws > 1:
        import torch.distributed as dist
        cs = checksum.reshape(1).to("cuda" if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(cs)
        checksum = cs[0]
    checksum = float(checksum)
    algo = 8.0 * n * n * sum(4.0 ** -l for l in range(levels))
    gbs_per_gpu = algo / ws / (ms * 1e-3) / 1e9
    sp.close()
    del out
    return {"workload": f"configs[3]: cdf97 monolithic_star {levels}-level forward pyramid, "
                        f"{n}x{n} float32, periodic, {ws} row strip(s) of {n // ws} rows, "
                        "halo rows pushed per level over peer memory (CUDA IPC)",
            "value": n * n / (ms * 1e-3) / 1e9, "unit": "GPixel/s (input pixels)",
            "ms": ms, "ns_per_pixel": ms * 1e6 / (n * n), "scaling": "strong", "ranks": ws,
            "checksum": checksum,
            "algorithmic_bytes": algo, "hbm_gbs_per_gpu": gbs_per_gpu,
            "frac_per_gpu": gbs_per_gpu / peak}


def run_c5(args, wl, ws, rank, peak):
    """BASELINE configs[4]: 4096 images of 4096^2, cdf53 and cdf97
    monolithic_star 3-level forward, images sharded over ranks (no
    communication). A resident pool of distinct images is cycled: each rank's
    share is processed in batched launches of `chunk` images."""
    import torch
    total, n, levels = args.c5_images, 4096, 3
    mine = total // ws
    chunk = min(64, mine)
    pool = max(chunk, min(mine, args.c5_pool) // chunk * chunk)
    g = torch.Generator(device="cuda").manual_seed(5000 + rank)
    imgs = torch.rand((pool, n, n), device="cuda", generator=g)
    pyrs = torch.empty((pool, n * n), device="cuda")
    scratch = torch.empty(wl.lib().wl_pyramid_batch_scratch_elems(n, n, levels, chunk),
                          device="cuda")
    stream = torch.cuda.current_stream()
    res = {}
    for w in ("cdf53", "cdf97"):
        sch = wl.build_scheme("monolithic_star", w)

        def job():
            for c in range(mine // chunk):
                i = (c * chunk) % pool
                wl.multi_level_forward_batch(imgs[i:i + chunk], sch, levels,
                                             out=pyrs[i:i + chunk], scratch=scratch)
        job()
        torch.cuda.synchronize()
        res[w] = _timed(job, max(1, min(args.steps, 3)), ws, stream)
    del imgs, pyrs, scratch
    algo = 8.0 * n * n * sum(4.0 ** -l for l in range(levels)) * total
    out = {"workload": f"configs[4]: {total} images x {n}^2 float32, monolithic_star "
                       f"{levels}-level forward, cdf53 and cdf97; {mine} images per rank in "
                       f"batched launches of {chunk}; resident pool of {pool} distinct images "
                       "per rank cycled (pool > L2)", "scaling": "strong",
           "unit": "GPixel/s (input pixels, whole job)"}
    for w, ms in res.items():
        gbs = algo / ws / (ms * 1e-3) / 1e9
        out[w] = {"ms": ms, "value": total * n * n / (ms * 1e-3) / 1e9,
                  "ns_per_pixel": ms * 1e6 / (total * n * n), "hbm_gbs_per_gpu": gbs,
                  "frac_per_gpu": gbs / peak}
    out["value"] = 2 * total * n * n / (sum(res.values()) * 1e-3) / 1e9
    return out


def cpu_baseline(args, gpu_ms, c0_gpu_ms=None):
    """The unmodified reference (oracle/_ref) on this host at the FULL
    configs[1] size (n x n, float64) for the headline pair: cdf53 Monolithic
    and cdf97 Monolithic* forward (transform.cpp:163) + the reference inverse
    (transform.cpp:178), next to the GPU's isolated times of the same
    programs (same size, same input distribution); plus configs[0], the
    reference CLI's bench shape (1024^2 cdf53 Sweldens forward)."""
    try:
        import numpy as np
        ref, kind, cores = _ref_lib()
        n = args.size
        img = np.random.default_rng(12345).random((n, n))
        same, px, tot = {}, 0, 0.0
        for (w, s) in CPU_FULL:
            t0 = time.perf_counter()
            qd = ref.forward(img, w, s, "periodic", False)
            t1 = time.perf_counter()
            ref.inverse(qd, w, "periodic", False)
            t2 = time.perf_counter()
            del qd
            for d, t in (("fwd", t1 - t0), ("inv", t2 - t1)):
                key = f"{w}/{s}/{d}"
                g_ms = gpu_ms.get(key)
                same[key] = {"cpu_ms": round(1e3 * t, 1), "cpu_ns_per_px": round(1e9 * t / img.size, 2),
                             "gpu_ms": round(g_ms, 5) if g_ms else None,
                             "gpu_over_cpu": round(1e3 * t / g_ms, 1) if g_ms else None}
            px += 2 * img.size
            tot += t2 - t0
        # configs[0]: the reference CLI's bench shape (wavelift_main.cpp:236-272), 1024^2
        # cdf53 Sweldens forward, median of 5 runs
        im0 = np.random.default_rng(1).random((1024, 1024))
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            ref.forward(im0, "cdf53", "sweldens", "periodic", False)
            ts.append(time.perf_counter() - t0)
        t0s = statistics.median(ts)
        c0 = {"workload": "configs[0]: cdf53 sweldens single-level forward, 1024x1024 "
                          "(reference float64 on the host cores vs the GPU float32, isolated)",
              "cpu_ms": round(1e3 * t0s, 2), "cpu_ns_per_px": round(1e9 * t0s / im0.size, 2),
              "gpu_ms": round(c0_gpu_ms, 5) if c0_gpu_ms else None,
              "gpu_over_cpu": round(1e3 * t0s / c0_gpu_ms, 1) if c0_gpu_ms else None}
        return {"value": px / tot / 1e9, "unit": "GPixel/s", "cores": cores, "kind": kind,
                "configs0": c0,
                "ns_per_pixel": 1e9 * tot / px, "seconds": round(tot, 2),
                "sample": f"{n}x{n} float64 (the full configs[1] size), uniform[0,1) numpy seed "
                          f"12345: cdf53 monolithic and cdf97 monolithic_star, forward + "
                          f"reference inverse, 1 pass each, periodic, {cores} threads",
                "same_config": same}
    except Exception as e:  # report, never fake
        return {"value": None, "unit": "GPixel/s", "cores": None, "kind": "unavailable",
                "sample": f"error: {e}"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--size", type=int, default=SIZE)
    ap.add_argument("--ref-rows", type=int, default=256,
                    help="reference arm: rows of the 8192-wide band timed per step")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-c3", dest="c3", action="store_false")
    ap.add_argument("--no-c4", dest="c4", action="store_false")
    ap.add_argument("--no-c5", dest="c5", action="store_false")
    ap.add_argument("--c4-size", type=int, default=32768)
    ap.add_argument("--c5-images", type=int, default=4096)
    ap.add_argument("--c5-pool", type=int, default=256)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-unaligned", dest="unaligned", action="store_false")
    ap.add_argument("--no-dd137", dest="dd137", action="store_false")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
