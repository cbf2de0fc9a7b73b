"""Dev tool: the fused kernels against the split kernels on a config (timing and agreement)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1210_0084_b200 import api
from synth.configs import CONFIGS

cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
n = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.n
batch = int(sys.argv[3]) if len(sys.argv) > 3 else cfg.batch
torch.manual_seed(0)
x = torch.randn(batch, n, device="cuda") * 0.1
plans, outs = {}, {}
for fused in (0, 1):
    os.environ["SLICQ_FUSED"] = str(fused)
    plans[fused] = api.plan_for_config(cfg)
def timeit(fn, it=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it
for fused, plan in plans.items():
    c = plan.forward(x); y = plan.inverse(c, n); torch.cuda.synchronize()
    tf = timeit(lambda: plan.forward(x, out=c))
    ti = timeit(lambda: plan.inverse(c, n, out=y))
    err = (torch.linalg.vector_norm(y - x) / torch.linalg.vector_norm(x)).item()
    outs[fused] = (c.clone(), y.clone())
    print(f"fused={fused}: fwd {tf:.3f} ms  inv {ti:.3f} ms  recon {err:.2e}  launches f/i "
          f"{plan.kernel_launches('forward', c.shape[1], batch)}/{plan.kernel_launches('inverse', c.shape[1], batch)}", flush=True)
c0, c1 = outs[0][0], outs[1][0]
d = torch.linalg.vector_norm((c1 - c0).reshape(-1, c0.shape[-1]), dim=1)
r = torch.linalg.vector_norm(c0.reshape(-1, c0.shape[-1]), dim=1)
print(f"coeff max per-slice rel diff fused vs split: {(d / r.clamp_min(1e-30)).max().item():.3e}")
