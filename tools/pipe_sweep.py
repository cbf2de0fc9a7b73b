"""Dev tool: split-path timing vs chunk count (SLICQ_PIPE_PARTS; staging per chunk ~ units/parts)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1210_0084_b200 import api
from synth.configs import CONFIGS
cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
parts = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "4,16,32,48,64,96").split(",")]
n, batch = cfg.n, cfg.batch
x = torch.randn(batch, n, device="cuda") * 0.1
os.environ["SLICQ_FUSED"] = "0"
for P in parts:
    os.environ["SLICQ_PIPE_PARTS"] = str(P)
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
    print(f"parts={P:4d} fwd {res[0]:.3f} inv {res[1]:.3f} ms launches {plan.kernel_launches('forward', c.shape[1], batch)}", flush=True)
    plan.close(); del plan
