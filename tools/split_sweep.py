"""Dev tool: split-path forward / inverse timing for env variants (semicolon-separated)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1210_0084_b200 import api
from synth.configs import CONFIGS
cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
variants = sys.argv[2].split(";") if len(sys.argv) > 2 else [""]
n, batch = cfg.n, cfg.batch
x = torch.randn(batch, n, device="cuda") * 0.1
ref = None
for v in variants:
    for kv in [k for k in os.environ if k.startswith("SLICQ_")]:
        os.environ.pop(kv)
    os.environ["SLICQ_BAND"] = "0"
    for kv in filter(None, v.split(",")):
        k, val = kv.split("="); os.environ[k] = val
    plan = api.plan_for_config(cfg)
    c = plan.forward(x); y = plan.inverse(c, n); torch.cuda.synchronize()
    res = []
    for fn in (lambda: plan.forward(x, out=c), lambda: plan.inverse(c, n, out=y)):
        for _ in range(3): fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): fn()
        e1.record(); torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) / 10)
    if ref is None:
        ref = (c.clone(), y.clone()); dc = dy = 0.0
    else:
        dc = (c - ref[0]).abs().max().item(); dy = (y - ref[1]).abs().max().item()
    print(f"[{v or 'default'}] fwd {res[0]:.3f} inv {res[1]:.3f} ms  diff c {dc:.1e} y {dy:.1e}", flush=True)
    plan.close(); del plan
