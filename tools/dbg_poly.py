import ctypes, torch, sys
sys.path.insert(0,'.')
import paper_1605_00561_b200 as wl
for n in (1024, 2048, 4096, 8192):
    img = torch.rand((n, n), device="cuda")
    try:
        q = wl.forward(img, wl.build_scheme("polyphase", "cdf97"))
        torch.cuda.synchronize(); print(n, "fwd ok")
    except Exception as e:
        print(n, "fwd FAIL", e)
    try:
        q = wl.forward(img, wl.build_scheme("monolithic", "cdf97"))
        torch.cuda.synchronize(); print(n, "mono fwd ok")
    except Exception as e:
        print(n, "mono FAIL", e)
