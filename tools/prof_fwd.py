"""Dev tool for ncu: warm-up + one profiled call of one direction on a config (n samples)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1210_0084_b200 import api
from synth.configs import CONFIGS
cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 16 * 148 * 8192
direction = sys.argv[3] if len(sys.argv) > 3 else "forward"
plan = api.plan_for_config(cfg)
x = torch.randn(1, n, device="cuda") * 0.1
c = plan.forward(x); y = plan.inverse(c, n)
torch.cuda.synchronize()
if direction == "forward":
    plan.forward(x, out=c)
else:
    plan.inverse(c, n, out=y)
torch.cuda.synchronize()
print("ok", tuple(c.shape))
