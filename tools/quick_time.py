"""Quick kernel timing (dev tool): CUDA-event timing of forward/inverse on a config."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1210_0084_b200 import api
from synth.configs import CONFIGS
from synth.signals import random_signal

cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
n = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.n
batch = int(sys.argv[3]) if len(sys.argv) > 3 else cfg.batch
plan = api.plan_for_config(cfg)
x = torch.randn(batch, n, device="cuda") * 0.1
c = plan.forward(x); y = plan.inverse(c, n); torch.cuda.synchronize()
S = c.shape[1]
for name, fn in (("fwd", lambda: plan.forward(x, out=c)), ("inv", lambda: plan.inverse(c, n, out=y))):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    it = 10
    e0.record()
    for _ in range(it): fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / it
    L = plan.padded_length(n)
    byts = batch * (4 * L + 8 * S * plan.coeffs_per_slice)
    print(f"{name}: {ms:.3f} ms  {batch*n/ms/1e6:.2f} Gsamples/s  {byts/ms/1e6:.1f} GB/s  slices={S} batch={batch}")
err = (torch.linalg.vector_norm(y - x) / torch.linalg.vector_norm(x)).item()
print("roundtrip rel err", err)
