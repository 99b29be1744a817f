"""Small workload for compute-sanitizer racecheck/synccheck (all engines)."""
import sys, torch
sys.path.insert(0, '.')
import paper_1605_00561_b200 as wl
img = torch.rand((256, 512), device='cuda')
for eng in (0, 1):
    wl.set_engine(eng)
    for w in ('cdf53', 'cdf97'):
        for s in wl.SCHEMES:
            for b in ('periodic', 'symmetric'):
                q = wl.forward(img, wl.build_scheme(s, w), b)
                wl.inverse(q, w, b, scheme=s)
torch.cuda.synchronize()
print('done')
