"""Sweep staging chunk / tile sizes (env read at plan creation) for a config (dev tool)."""
import os, sys, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1210_0084_b200 import api
from synth.configs import CONFIGS
cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
n = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.n
batch = int(sys.argv[3]) if len(sys.argv) > 3 else cfg.batch
chunks = [int(v) for v in (sys.argv[4] if len(sys.argv) > 4 else "592,1184,2368,1000000").split(",")]
tiles = [int(v) for v in (sys.argv[5] if len(sys.argv) > 5 else "8,16,32").split(",")]
x = torch.randn(batch, n, device="cuda") * 0.1
for cu, t in itertools.product(chunks, tiles):
    os.environ["SLICQ_CHUNK_UNITS"] = str(cu); os.environ["SLICQ_TILE"] = str(t)
    plan = api.plan_for_config(cfg)
    c = plan.forward(x); y = plan.inverse(c, n); torch.cuda.synchronize()
    res = []
    for fn in (lambda: plan.forward(x, out=c), lambda: plan.inverse(c, n, out=y)):
        for _ in range(2): fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): fn()
        e1.record(); torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) / 5)
    print(f"chunk={cu:8d} tile={t:3d}  fwd {res[0]:.3f} ms  inv {res[1]:.3f} ms", flush=True)
    plan.close(); del plan
