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
             timed region.
* roofline   dominant kernel of the step (largest share of step time):
             algorithmic bytes = 8 B/pixel (one f32 read + one f32 write per
             pixel) / its CUDA-event launch time, against the
             measured HBM copy peak (MEASURED_PEAKS.json).
* c3         BASELINE.json configs[2]: cdf97 monolithic_star, 16384^2, fwd & inv.
* per_scheme GPix/s, ns/px and HBM fraction for each of the 40 programs.
* cpu_baseline  the unmodified reference (oracle/_ref, "reference") on the
             host cores, bounded sample (see its "sample").

`--impl reference` times the reference's CPU implementation of the same step
on a bounded 512^2 sample (rank 0 only under torchrun).
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


def run_reference(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import numpy as np
    from oracle.oracle import RefLib, Oracle
    n = args.ref_size
    try:
        ref = RefLib()
        kind = "reference"
    except FileNotFoundError:
        ref, kind = Oracle(), "port"
    img = np.random.default_rng(12345).random((n, n))
    cores = ref.worker_count() if kind == "reference" else 1
    for _ in range(args.warmup):
        reference_step_sample(ref, img)
    times, px = [], 0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        px = reference_step_sample(ref, img)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    gpix = px * args.steps / tot / 1e9
    sample = (f"{n}x{n} float64 uniform[0,1) (mt-free numpy seed 12345), every scheme x "
              f"{{cdf53,cdf97}} forward + reference inverse per step, periodic, no scaling, "
              f"WAVELIFT_THREADS={os.environ.get('WAVELIFT_THREADS', 'unset')} -> {cores} "
              f"worker threads")
    line = {"impl": "reference", "metric": METRIC, "value": gpix, "unit": "GPixel/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "ns_per_pixel": 1e9 * tot / (px * args.steps),
            "config": {"workload": f"configs[1] sample: {n}^2, all schemes x cdf53/cdf97, "
                                   "fwd + inv", "size": n, "parallelism": "host threads"},
            "cpu_baseline": {"value": gpix, "unit": "GPixel/s", "cores": cores, "kind": kind,
                             "sample": sample},
            "e2e": {"value": gpix, "unit": "GPixel/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------- GPU arm
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
    programs = [(w, s) for w in WAVELETS for s in SCHEMES]
    schemes = {(w, s): wl.build_scheme(s, w) for (w, s) in programs}
    stream = torch.cuda.current_stream()

    def step(events=None):
        for i, (w, s) in enumerate(programs):
            if events is not None:
                events[4 * i].record(stream)
            wl.forward(img, schemes[(w, s)], "periodic", False, out=q)
            if events is not None:
                events[4 * i + 1].record(stream)
                events[4 * i + 2].record(stream)
            wl.inverse(q, w, "periodic", False, scheme=s, out=rec)
            if events is not None:
                events[4 * i + 3].record(stream)

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
        start.record(stream)
        for _ in range(args.steps):
            step()
        stop.record(stream)
        torch.cuda.synchronize()
        barrier(ws)
    launches = wl.launch_count() - n0
    ms = start.elapsed_time(stop) / args.steps
    ms = barrier_max(ms, ws)
    px_step = 2 * len(programs) * n * n
    value = ws * px_step / (ms * 1e-3) / 1e9

    # ---- per-kernel times (CUDA events on the launching stream), separate pass
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4 * len(programs))]
    per = {}
    reps = max(1, min(args.steps, 5))
    acc = [0.0] * (2 * len(programs))
    for _ in range(reps):
        step(ev)
        torch.cuda.synchronize()
        for i in range(2 * len(programs)):
            acc[i] += ev[2 * i].elapsed_time(ev[2 * i + 1])
    algo_bytes = 8.0 * n * n
    for i, (w, s) in enumerate(programs):
        for d, name in ((0, "fwd"), (1, "inv")):
            t = acc[2 * i + d] / reps
            gbs = algo_bytes / (t * 1e-3) / 1e9
            per[f"{w}/{s}/{name}"] = {"ms": round(t, 5), "gpix_s": round(n * n / t / 1e6, 2),
                                      "ns_per_px": round(t * 1e6 / (n * n), 6),
                                      "hbm_gbs": round(gbs, 1), "frac": round(gbs / peak, 4)}
    # dominant kernel = largest share of the step, per actual kernel: the
    # Convolution scheme's inverse is the reference inverse (the Sweldens
    # inverse kernel), so both programs' launches count for that kernel
    def kernel_of(prog):
        w_, s_, d_ = prog.split("/")
        return f"{w_}/sweldens/inv" if (s_ == "convolution" and d_ == "inv") else prog
    share = {}
    for k, v in per.items():
        share[kernel_of(k)] = share.get(kernel_of(k), 0.0) + v["ms"]
    dom = max(share, key=share.get)
    dom_t = per[dom]["ms"]
    step_sum = sum(v["ms"] for v in per.values())
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic_r01.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(dom)
        except Exception:
            traffic = None
    # FP32 side of the same kernel: MACs per quad (count_macs, schemes.cpp:176)
    # -> FMA per pixel = MACs / 4; nominal FP32 peak 148 SMs x 128 FMA/clk x
    # 2 FLOP x max SM clock.
    dw, ds, dd = dom.split("/")
    macs = schemes[(dw, ds)].info(0 if dd == "fwd" or ds == "convolution" else 1)["macs"]
    fp32_peak = 148 * 128 * 2 * 1.965e9 / 1e12
    fp32 = 2.0 * macs / 4.0 * n * n / (dom_t * 1e-3) / 1e12
    roofline = {"bound": "hbm", "kernel": dom, "achieved": per[dom]["hbm_gbs"], "peak": peak,
                "peak_source": peak_src, "unit": "GB/s", "frac": per[dom]["frac"],
                "traffic": traffic, "share_of_step": round(share[dom] / step_sum, 4),
                "launches_per_step": sum(1 for k in per if kernel_of(k) == dom),
                "algorithmic_bytes_per_launch": algo_bytes,
                "fp32": {"fma_per_px": macs / 4.0, "achieved_tflops": round(fp32, 2),
                         "peak_tflops_nominal": round(fp32_peak, 1),
                         "frac": round(fp32 / fp32_peak, 4)}}

    # ---- C3 headline: cdf97 monolithic_star, 16384^2 (configs[2])
    c3 = None
    if args.c3:
        big = torch.rand((C3, C3), device=dev, generator=g, dtype=torch.float32)
        qb = torch.empty((4, C3 // 2, C3 // 2), device=dev, dtype=torch.float32)
        rb = torch.empty_like(big)
        c3 = {}
        for sname in ("monolithic_star", "monolithic", "sweldens"):
            sch = wl.build_scheme(sname, "cdf97")
            for _ in range(3):
                wl.forward(big, sch, out=qb)
                wl.inverse(qb, "cdf97", scheme=sname, out=rb)
            e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            tf = ti = 0.0
            r = 10
            for _ in range(r):
                e[0].record(stream)
                wl.forward(big, sch, out=qb)
                e[1].record(stream)
                wl.inverse(qb, "cdf97", scheme=sname, out=rb)
                e[2].record(stream)
                torch.cuda.synchronize()
                tf += e[0].elapsed_time(e[1])
                ti += e[1].elapsed_time(e[2])
            for name, t in (("fwd", tf / r), ("inv", ti / r)):
                gbs = 8.0 * C3 * C3 / (t * 1e-3) / 1e9
                c3[f"cdf97/{sname}/{name}"] = {
                    "ms": round(t, 4), "gpix_s": round(C3 * C3 / t / 1e6, 1),
                    "ns_per_px": round(t * 1e6 / (C3 * C3), 6), "hbm_gbs": round(gbs, 1),
                    "frac": round(gbs / peak, 4)}
        del big, qb, rb

    # ---- e2e through the public API with pinned host buffers
    e2e = None
    if args.e2e_steps > 0:
        # The reference-facing call shape: forward(const Image&) /
        # inverse(const QuadGrid&) on HOST buffers (wl_dwt2_forward_host /
        # wl_dwt2_inverse_host: row-chunk pipeline, H2D/kernels/D2H overlap).
        h_img = torch.empty((n, n), dtype=torch.float32, pin_memory=True)
        h_img.copy_(img.cpu())
        h_q = torch.empty((4, n // 2, n // 2), dtype=torch.float32, pin_memory=True)
        h_rec = torch.empty((n, n), dtype=torch.float32, pin_memory=True)

        def e2e_step():
            for (w, s) in programs:
                wl.forward_host(h_img, schemes[(w, s)], out=h_q)    # host image -> host planes
                wl.inverse_host(h_q, w, scheme=s, out=h_rec)        # host planes -> host image

        e2e_step()
        torch.cuda.synchronize()
        barrier(ws)
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()  # synchronous calls: results are in host memory on return
        ems = barrier_max((time.perf_counter() - t0) * 1e3 / args.e2e_steps, ws)
        bytes_img = 4 * n * n
        e2e = {"value": ws * px_step / (ems * 1e-3) / 1e9, "unit": "GPixel/s",
               "ms_per_step": ems, "h2d_bytes_per_step": 2 * len(programs) * bytes_img,
               "d2h_bytes_per_step": 2 * len(programs) * bytes_img,
               "steps": args.e2e_steps,
               "api": "forward_host / inverse_host (pinned host float32 buffers; wall clock "
                      "around synchronous calls); byte counts are the image/plane tensors, "
                      "the strip halo rows add <=1.2% H2D"}

    c4 = run_c4(args, wl, ws, rank, peak) if args.c4 else None
    c5 = run_c5(args, wl, ws, rank, peak) if args.c5 else None

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        cpu = cpu_baseline(args)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "GPixel/s", "n_gpus": ws,
                "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f32", "data": "synthetic",
                "ns_per_pixel": ms * 1e6 / px_step,
                "config": {"workload": f"configs[1]: every scheme x {{cdf53, cdf97}}, "
                                       f"single-level forward + that scheme's inverse, "
                                       f"{n}x{n} float32 per rank, periodic, no scaling",
                           "size": n, "programs": len(programs),
                           "pixels_per_step_per_rank": px_step,
                           "l2": "inputs (256 MiB) larger than L2 (126 MB); no flush",
                           "parallelism": f"independent images, {ws} rank(s)"},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches, "gpu_launches_per_step": launches / args.steps,
                "clocks": clk.summary(), "c3": c3, "c4": c4, "c5": c5, "per_scheme": per}
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


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
    g = torch.Generator(device="cuda").manual_seed(4000 + rank)
    sp.input.copy_(torch.rand(sp.input.shape, device="cuda", generator=g))
    out = torch.empty(sp.slice_elems(), device="cuda")
    stream = torch.cuda.current_stream()
    torch.cuda.synchronize()
    barrier(ws)  # every rank connected and idle before the first halo wait
    for _ in range(3):
        sp.forward(out)
    torch.cuda.synchronize()
    ms = _timed(lambda: sp.forward(out), max(args.steps, 5), ws, stream)
    sp.check()
    algo = 8.0 * n * n * sum(4.0 ** -l for l in range(levels))
    gbs_per_gpu = algo / ws / (ms * 1e-3) / 1e9
    sp.close()
    del out
    return {"workload": f"configs[3]: cdf97 monolithic_star {levels}-level forward pyramid, "
                        f"{n}x{n} float32, periodic, {ws} row strip(s) of {n // ws} rows, "
                        "halo rows pushed per level over peer memory (CUDA IPC)",
            "value": n * n / (ms * 1e-3) / 1e9, "unit": "GPixel/s (input pixels)",
            "ms": ms, "ns_per_pixel": ms * 1e6 / (n * n), "scaling": "strong",
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


def cpu_baseline(args):
    """The unmodified reference (oracle/_ref) on this host: bounded sample."""
    try:
        import numpy as np
        from oracle.oracle import Oracle, RefLib
        try:
            ref, kind = RefLib(), "reference"
        except FileNotFoundError:
            ref, kind = Oracle(), "port"
        n = args.ref_size
        img = np.random.default_rng(12345).random((n, n))
        t0 = time.perf_counter()
        px = reference_step_sample(ref, img)
        dt = time.perf_counter() - t0
        cores = ref.worker_count() if kind == "reference" else 1
        return {"value": px / dt / 1e9, "unit": "GPixel/s", "cores": cores, "kind": kind,
                "ns_per_pixel": 1e9 * dt / px, "seconds": dt,
                "sample": f"{n}x{n} float64, every scheme x {{cdf53,cdf97}} forward + "
                          f"reference inverse (1 pass each), periodic, {cores} threads"}
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
    ap.add_argument("--ref-size", type=int, default=512)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-c3", dest="c3", action="store_false")
    ap.add_argument("--no-c4", dest="c4", action="store_false")
    ap.add_argument("--no-c5", dest="c5", action="store_false")
    ap.add_argument("--c4-size", type=int, default=32768)
    ap.add_argument("--c5-images", type=int, default=4096)
    ap.add_argument("--c5-pool", type=int, default=256)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
