# cdf97 direct-load forwards: fewer warps per CTA, more CTAs per SM (8190^2)
mkdir -p gpurun_out
cat > /tmp/ud.py <<'PY'
import torch, sys, os
sys.path.insert(0, os.getcwd())
import paper_1605_00561_b200 as wl
n = 8190
img = torch.rand((n, n), device="cuda")
for w in ("cdf97", "cdf53"):
    for s in wl.SCHEMES[:9]:
        sch = wl.build_scheme(s, w)
        q = wl.forward(img, sch)
        for _ in range(3): wl.forward(img, sch, out=q)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            torch.cuda._sleep(5_000_000)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10): wl.forward(img, sch, out=q)
            e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1) / 10)
        ts.sort()
        print(os.environ.get("WL_LIB", "base")[-10:], n, w, s, f"{ts[2]:.4f}")
PY
for i in 1 2; do for t in base n5m3 n6m3 n4m4; do
  if [ $t = base ]; then L=paper_1605_00561_b200/libwavelift_b200.so; else L=paper_1605_00561_b200/libwavelift_b200_$t.so; fi
  WL_LIB=$L python /tmp/ud.py; done; done > gpurun_out/g15_ab.txt 2>&1
