"""Dev probe for compute-sanitizer: small forward/inverse/range/process_host calls over the
kernel families (2N = 4096 .. 131072, raster modes, ragged lengths)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1210_0084_b200 import api
cases = [(44100, 65.4, 22050, 12, 16384, 2048, 0, 70001, 2), (44100, 32.7, 22050, 48, 32768, 4096, 1, 100000, 1),
         (44100, 55, 22050, 24, 16384, 2048, 2, 40000, 1), (44100, 100, 22050, 12, 4096, 512, 0, 9000, 3),
         (44100, 50, 22050, 48, 65536, 4096, 0, 140000, 1), (44100, 60, 22050, 96, 131072, 2000, 0, 262144, 1)]
for fs, fmin, fmax, B, sl, tr, ra, n, batch in cases:
    p = api.Plan(fs, fmin, fmax, B, sl, tr, ra)
    x = torch.randn(batch, n, device="cuda") * 0.1
    c = p.forward(x)
    y = p.inverse(c, n)
    S = c.shape[1]
    half = S // 2
    halo = p.halo + (p.halo & 1)
    N = p.N
    xl = torch.zeros(batch, halo + (S - half) * N, device="cuda")
    cl = p.forward_range(xl, halo, half, S - half, S)
    yl, sp = p.inverse_range(cl, half, S - half, S, halo)
    torch.cuda.synchronize()
    print("ok", sl, ra, tuple(c.shape), float((y - x).norm() / x.norm()), flush=True)
p = api.Plan(44100, 65.4, 22050, 12, 16384, 2048, 0)
xh = torch.randn(1, 200001).mul_(0.1).pin_memory()
yh = api.process_host(p, xh, pieces=4)
torch.cuda.synchronize()
print("process_host ok", flush=True)
