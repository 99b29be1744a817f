import sys, torch
sys.path.insert(0, '.')
import paper_1605_00561_b200 as wl
img = torch.rand((512, 768), device='cuda')
for w in ['cdf53', 'cdf97']:
    for s in wl.SCHEMES[:9]:
        wl.set_engine(2)
        q = wl.forward(img, wl.build_scheme(s, w)); r = wl.inverse(q, w, scheme=s)
        wl.set_engine(1)
        q1 = wl.forward(img, wl.build_scheme(s, w)); r1 = wl.inverse(q1, w, scheme=s)
        torch.cuda.synchronize()
        print(w, s, 'fwd diff', (q - q1).abs().max().item(), 'inv diff', (r - r1).abs().max().item(), 'PR', (r - img).abs().max().item(), flush=True)
