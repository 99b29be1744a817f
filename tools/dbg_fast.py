import sys, torch
sys.path.insert(0, '.')
import paper_1605_00561_b200 as wl
for rep in range(4):
    for wavelet in ('cdf53', 'cdf97'):
        g = torch.Generator(device="cuda").manual_seed(5)
        img = torch.rand((2048, 4096), device="cuda", generator=g)
        for scheme in wl.SCHEMES[:9]:
            for b in ('periodic', 'symmetric'):
                q = wl.forward(img, wl.build_scheme(scheme, wavelet), b, True)
                rec = wl.inverse(q, wavelet, b, True, scheme=scheme)
                d = (rec - img).abs()
                err = d.max().item()
                if err > 1e-4 and not (b == 'symmetric' and scheme.startswith('polyphase')):
                    bad = (d > 1e-4).nonzero()
                    wl.set_engine(1)
                    q1 = wl.forward(img, wl.build_scheme(scheme, wavelet), b, True)
                    wl.set_engine(0)
                    dq = (q - q1).abs(); bq = (dq > 1e-5).nonzero()
                    print(rep, wavelet, scheme, b, 'err', err, 'n', bad.shape[0], 'rows', bad[:, 0].min().item(), bad[:, 0].max().item(), 'cols', bad[:, 1].min().item(), bad[:, 1].max().item(),
                          '| fwd bad n', bq.shape[0], (bq.min(0).values.tolist(), bq.max(0).values.tolist()) if bq.shape[0] else '', flush=True)
print('end')
