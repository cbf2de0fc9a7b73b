"""Dev probe: api.process_host round-trip time vs the number of slice ranges (cfg4)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1210_0084_b200 import api
from synth.configs import CONFIGS
cfg = CONFIGS[4]
plan = api.plan_for_config(cfg)
n = cfg.n
x = torch.randn(1, n).mul_(0.1).pin_memory()
y = torch.empty(1, n, pin_memory=True)
for pieces in [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "8,16,32,64").split(",")]:
    for _ in range(2): api.process_host(plan, x, y, pieces=pieces)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): api.process_host(plan, x, y, pieces=pieces)
    e1.record(); torch.cuda.synchronize()
    print(f"pieces={pieces}: {e0.elapsed_time(e1)/5:.2f} ms", flush=True)
