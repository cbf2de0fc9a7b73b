"""Dev tool: forward/inverse time and agreement of plan variants selected by an env switch.

    python tools/variant_check.py CFG VAR V0,V1,...   e.g.  4 SLICQ_CLUSTER 0,4,8,16
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1210_0084_b200 import api
from synth.configs import CONFIGS

cfg = CONFIGS[int(sys.argv[1])]
var, vals = sys.argv[2], sys.argv[3].split(",")
n, batch = cfg.n, cfg.batch
torch.manual_seed(0)
x = torch.randn(batch, n, device="cuda") * 0.1


def timeit(fn, it=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it


ref = None
for v in vals:
    os.environ[var] = v
    plan = api.plan_for_config(cfg)
    c = plan.forward(x); y = plan.inverse(c, n); torch.cuda.synchronize()
    tf = timeit(lambda: plan.forward(x, out=c))
    ti = timeit(lambda: plan.inverse(c, n, out=y))
    err = (torch.linalg.vector_norm(y - x) / torch.linalg.vector_norm(x)).item()
    if ref is None:
        ref = c.clone()
        dmax = 0.0
    else:
        d = torch.linalg.vector_norm((c - ref).reshape(-1, c.shape[-1]), dim=1)
        r = torch.linalg.vector_norm(ref.reshape(-1, c.shape[-1]), dim=1)
        dmax = (d / r.clamp_min(1e-30)).max().item()
    print(f"{var}={v}: fwd {tf:.3f} ms  inv {ti:.3f} ms  recon {err:.2e}  "
          f"max per-slice rel diff vs {vals[0]}: {dmax:.2e}", flush=True)
    del plan
