"""Dev tool: full-length CQ-NSGT throughput (slicq_nsgt_forward / inverse) for a batch of
signals of one length L (the paper's CQ-NSGT comparison scale, NEXT-1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1210_0084_b200 import api
CASES = ((16384, 1024, 24, 50.0), (131072, 128, 96, 60.0), (2 ** 18, 64, 48, 50.0),
         (2 ** 20, 16, 48, 50.0), (2 ** 21, 8, 96, 60.0), (2 ** 22, 4, 96, 60.0),
         (2 ** 22, 4, 48, 60.0))
if len(sys.argv) > 1:
    CASES = [c for c in CASES if c[0] == int(sys.argv[1])][:1]
for L, B, bpo, fmin in CASES:
    plan = api.Plan(44100.0, fmin, 22050.0, bpo, L, 64, 0)
    x = torch.randn(B, L, device="cuda") * 0.1
    c = plan.nsgt_forward(x)
    y = plan.nsgt_inverse(c, L)
    torch.cuda.synchronize()
    res = []
    for fn in (lambda: plan.nsgt_forward(x, out=c), lambda: plan.nsgt_inverse(c, L, out=y)):
        for _ in range(3): fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): fn()
        e1.record(); torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) / 10)
    err = ((y - x).norm() / x.norm()).item()
    print(f"L={L} batch={B}: forward {res[0]:.3f} ms ({B*L/res[0]/1e6:.1f} G samples/s), "
          f"inverse {res[1]:.3f} ms, reconstruction {err:.1e}", flush=True)
