"""Dev tool: fused masked inverse vs separate mask + inverse (cfg4)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1210_0084_b200 import api
from synth.configs import CONFIGS
cfg = CONFIGS[4]
plan = api.plan_for_config(cfg)
n = cfg.n
x = torch.randn(1, n, device="cuda") * 0.1
c = plan.forward(x)
m = torch.rand(c.shape, device="cuda")
y = plan.inverse(c, n)
def t(fn, it=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it
print(f"inverse {t(lambda: plan.inverse(c, n, out=y)):.3f} ms  "
      f"fused masked {t(lambda: plan.inverse(c, n, out=y, mask=m)):.3f} ms  "
      f"separate mask + inverse {t(lambda: plan.inverse(api.apply_mask(plan, c, m), n, out=y)):.3f} ms")
