"""Dev tool: forward timing and agreement for env-selected paths (SLICQ_RING / SLICQ_FUSED)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1210_0084_b200 import api
from synth.configs import CONFIGS
cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
n = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.n
batch = int(sys.argv[3]) if len(sys.argv) > 3 else cfg.batch
variants = sys.argv[4].split(";") if len(sys.argv) > 4 else ["SLICQ_FUSED=0", "SLICQ_RING=0", ""]
torch.manual_seed(0)
x = torch.randn(batch, n, device="cuda") * 0.1
ref = None
for v in variants:
    for kv in [k for k in os.environ if k.startswith("SLICQ_")]:
        os.environ.pop(kv, None)
    for kv in filter(None, v.split(",")):
        k, val = kv.split("=")
        os.environ[k] = val
    plan = api.plan_for_config(cfg)
    c = plan.forward(x); torch.cuda.synchronize()
    for _ in range(3): plan.forward(x, out=c)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): plan.forward(x, out=c)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    if ref is None:
        ref = c.clone(); diff = 0.0
    else:
        d = torch.linalg.vector_norm((c - ref).reshape(-1, c.shape[-1]), dim=1)
        r = torch.linalg.vector_norm(ref.reshape(-1, c.shape[-1]), dim=1)
        diff = (d / r.clamp_min(1e-30)).max().item()
    print(f"[{v or 'default'}] fwd {ms:.3f} ms  launches {plan.kernel_launches('forward', c.shape[1], batch)}  maxdiff {diff:.2e}", flush=True)
    plan.close()
