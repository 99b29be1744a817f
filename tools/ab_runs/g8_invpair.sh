# direct-load inverses: float2/float4 image-row stores vs element-wise, 8190^2 / 8194^2; parity tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity_large.py tests/test_gpu_batch_strip.py -q -k "unaligned or direct" > gpurun_out/g8_tests.log 2>&1; echo rc=$? >> gpurun_out/g8_tests.log
cat > /tmp/uinv.py <<'PY'
import torch, sys, os
sys.path.insert(0, os.getcwd())
import paper_1605_00561_b200 as wl
for n in (8190, 8194):
    img = torch.rand((n, n), device="cuda")
    for w in ("cdf53", "cdf97"):
        for s in wl.SCHEMES[:9]:
            sch = wl.build_scheme(s, w)
            q = wl.forward(img, sch)
            rec = wl.inverse(q, w, scheme=s)
            for _ in range(3): wl.inverse(q, w, scheme=s, out=rec)
            torch.cuda.synchronize()
            ts = []
            for _ in range(5):
                torch.cuda._sleep(5_000_000)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(10): wl.inverse(q, w, scheme=s, out=rec)
                e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1) / 10)
            ts.sort()
            print(os.environ.get("WL_LIB", "base")[-10:], n, w, s, f"{ts[2]:.4f}")
PY
for i in 1 2; do python /tmp/uinv.py; WL_LIB=paper_1605_00561_b200/libwavelift_b200_noinvp.so python /tmp/uinv.py; done > gpurun_out/g8_ab.txt 2>&1
