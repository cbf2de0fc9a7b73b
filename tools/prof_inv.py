"""Dev tool for ncu: warm-up + one profiled inverse on a config (n samples, batch)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1210_0084_b200 import api
from synth.configs import CONFIGS
cfg = CONFIGS[int(sys.argv[1])]
n = int(sys.argv[2]); batch = int(sys.argv[3])
plan = api.plan_for_config(cfg)
x = torch.randn(batch, n, device="cuda") * 0.1
c = plan.forward(x); y = plan.inverse(c, n); torch.cuda.synchronize()
plan.inverse(c, n, out=y); torch.cuda.synchronize()
print("ok", tuple(c.shape))
