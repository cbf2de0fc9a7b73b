"""Dev check: process_host (host round trip over slice ranges) vs the device path on cfg4."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1210_0084_b200 import api
from synth.configs import CONFIGS
from synth.signals import make_signal
cfg = CONFIGS[4]
plan = api.plan_for_config(cfg)
x = make_signal(4)
n = x.shape[1]
xh = torch.from_numpy(x).pin_memory()
yh = torch.empty_like(xh).pin_memory()
N = plan.N
for rep in range(2):
    api.process_host(plan, xh, yh, pieces=32)
    torch.cuda.synchronize()
    y = yh.numpy()
    err = np.abs(y - x[0] if x.ndim == 1 else y - x)
    bad = np.nonzero(err[0] > 1e-3)[0]
    print(rep, "rel", np.linalg.norm(y - x) / np.linalg.norm(x), "bad samples", bad.size,
          "first/last", (bad[:3], bad[-3:]) if bad.size else None, flush=True)
    if bad.size:
        sl = bad // N
        u, cnt = np.unique(sl, return_counts=True)
        print("  slices with errors:", u.size, "first:", list(zip(u[:8].tolist(), cnt[:8].tolist())))
        off = bad % N
        print("  offset-in-hop histogram (8 bins of N/8):", np.histogram(off, bins=8, range=(0, N))[0].tolist())
        print("  ratio y/x at bad:", (y[0, bad[:5]] / x[0, bad[:5]]).tolist())
yd = plan.inverse(plan.forward(xh.cuda()), n).cpu().numpy()
print("device path rel", np.linalg.norm(yd - x) / np.linalg.norm(x))
print("N", plan.N, "S", plan.num_slices(n))
key = [k for k in plan._ws if k[1] == "process_host"][0]
ws = plan._ws[key]
import ctypes
from paper_1210_0084_b200._lib import lib
nb = ws.numel() * 4
wsb = ws.view(torch.int32)
# counters: at the start of the range workspace (ExecLayout.ws offset); find via size: the range
# workspace is the tail of the buffer, its first nsmax*B ints are the counters
rws_bytes = int(lib().slicq_workspace_bytes(plan._h, 800, 1))
print("total ws bytes", nb)
for P in (2, 4, 8, 32):
    y2 = api.process_host(plan, xh, pieces=P)
    torch.cuda.synchronize()
    e = np.linalg.norm(y2.numpy() - x) / np.linalg.norm(x)
    print("pieces", P, "rel err", e, flush=True)
