# split-row TMA forwards for unaligned shapes: parity tests + bench (unaligned section) + A/B vs direct
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity_large.py -q -k "unaligned or split or direct" > gpurun_out/g4_tests.log 2>&1; echo rc=$? >> gpurun_out/g4_tests.log
cat > /tmp/ua.py <<'PY'
import torch, sys, os
sys.path.insert(0, os.getcwd())
import paper_1605_00561_b200 as wl
for n in (8190, 8194):
    img = torch.rand((n, n), device="cuda")
    for w, s in (("cdf53", "monolithic"), ("cdf97", "monolithic_star"), ("cdf97", "sweldens")):
        sch = wl.build_scheme(s, w)
        q = wl.forward(img, sch)
        for _ in range(3): wl.forward(img, sch, out=q)
        torch.cuda.synchronize()
        ts = []
        for _ in range(7):
            torch.cuda._sleep(5_000_000)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10): wl.forward(img, sch, out=q)
            e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1) / 10)
        ts.sort()
        ms = ts[3]
        print(os.environ.get("WL_SPLIT", "1"), n, w, s, f"{ms:.4f} ms", f"{2*n*n*4/ms/1e6:.0f} GB/s", f"{2*n*n*4/ms/1e6/6491.8:.3f}")
PY
for i in 1 2; do python /tmp/ua.py; WL_SPLIT=0 python /tmp/ua.py; done > gpurun_out/g4_ab.txt 2>&1
