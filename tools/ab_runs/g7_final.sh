# cdf53 direct-load realigned stores: A/B over all cdf53 schemes at 8190^2, full GPU tests, bench
mkdir -p gpurun_out
cat > /tmp/ua53.py <<'PY'
import torch, sys, os
sys.path.insert(0, os.getcwd())
import paper_1605_00561_b200 as wl
n = 8190
img = torch.rand((n, n), device="cuda")
for s in wl.SCHEMES[:9]:
    sch = wl.build_scheme(s, "cdf53")
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
    print(os.environ.get("WL_LIB", "base")[-9:], n, "cdf53", s, f"{ts[3]:.4f} ms")
PY
for i in 1 2; do python /tmp/ua53.py; WL_LIB=paper_1605_00561_b200/libwavelift_b200_noral.so python /tmp/ua53.py; done > gpurun_out/g7_ab.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g7_gputest.log 2>&1; echo rc=$? >> gpurun_out/g7_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g7_smoke.log 2>&1
timeout 400 python bench.py > gpurun_out/g7_bench.json 2> gpurun_out/g7_bench.err
