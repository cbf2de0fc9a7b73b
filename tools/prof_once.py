"""Dev tool for ncu: warm-up + one forward and one inverse launch on a config (n samples)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1210_0084_b200 import api
from synth.configs import CONFIGS
cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4 * 148 * 8192
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 1
plan = api.plan_for_config(cfg)
x = torch.randn(batch, n, device="cuda") * 0.1
c = plan.forward(x); y = plan.inverse(c, n)     # warm-up (2 launches)
plan.forward(x, out=c); plan.inverse(c, n, out=y)  # profiled
torch.cuda.synchronize()
print("ok", tuple(c.shape))
