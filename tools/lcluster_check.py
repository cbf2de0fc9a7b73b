"""2N = 131072: the 16-CTA cluster slice FFT (SLICQ_LCLUSTER=1) against the split column / row
kernels (=0): bit-identical coefficients and output, plus timing of both (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1210_0084_b200 import api
from synth.configs import CONFIGS
cfg = CONFIGS[5]
batch = int(sys.argv[1]) if len(sys.argv) > 1 else 16
n = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.n
torch.manual_seed(0)
x = torch.randn(batch, n, device="cuda") * 0.1
res = {}
for flag in ("0", "3"):
    os.environ["SLICQ_LCLUSTER"] = flag
    plan = api.plan_for_config(cfg)
    c = plan.forward(x); y = plan.inverse(c, n); torch.cuda.synchronize()
    t = []
    for fn in (lambda: plan.forward(x, out=c), lambda: plan.inverse(c, n, out=y)):
        for _ in range(3): fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): fn()
        e1.record(); torch.cuda.synchronize()
        t.append(e0.elapsed_time(e1) / 10)
    res[flag] = (c.clone(), y.clone(), t, plan.kernel_launches("forward", c.shape[1], batch),
                 plan.kernel_launches("inverse", c.shape[1], batch))
    err = ((y - x).norm() / x.norm()).item()
    print(f"LCLUSTER={flag}: fwd {t[0]:.3f} ms inv {t[1]:.3f} ms  launches {res[flag][3]}/{res[flag][4]}  rt err {err:.2e}")
    plan.close()
c0, y0 = res["0"][:2]
c1, y1 = res["3"][:2]
print("coefficients identical:", torch.equal(c0, c1), " max diff", (c0 - c1).abs().max().item())
print("output identical:", torch.equal(y0, y1), " max diff", (y0 - y1).abs().max().item())
