import sys, torch
import paper_1605_00561_b200 as wl
wl.lib()
sch = wl.build_scheme(sys.argv[1] if len(sys.argv) > 1 else "sweldens", "cdf53")
img = torch.rand((64, 96), device="cuda")
q1 = wl.forward(img, sch); torch.cuda.synchronize(); print("single ok")
imgs = torch.rand((3, 64, 96), device="cuda")
q = wl.forward_batch(imgs, sch); torch.cuda.synchronize(); print("batch ok")
print(torch.equal(q[1], wl.forward(imgs[1], sch)))
