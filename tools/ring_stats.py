"""Dev tool: per-role busy / wait times of the forward ring kernel (SLICQ_RING_STATS=1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SLICQ_RING_STATS"] = "1"
import numpy as np, torch
from paper_1210_0084_b200 import api
from synth.configs import CONFIGS
cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
n = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.n
x = torch.randn(1, n, device="cuda") * 0.1
plan = api.plan_for_config(cfg)
c = plan.forward(x)
for _ in range(3): plan.forward(x, out=c)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); plan.forward(x, out=c); e1.record(); torch.cuda.synchronize()
print(f"fwd {e0.elapsed_time(e1):.3f} ms")
import ctypes
from paper_1210_0084_b200 import _lib
info = (ctypes.c_longlong * 8)()
fn = _lib.lib().slicq_debug_ring_info
fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
assert fn(plan._h, info) == 0
R, slot, nb, q, bt, nspec, soff, smem = list(info)
print(f"R={R} slot={slot} nb={nb} q={q} bt={bt} nspec={nspec} smem={smem}")
ws = list(plan._ws.values())[0]
wsb = ws.view(torch.uint8).flatten()
st = wsb[soff:soff + 1024 * 4 * 8].clone().view(torch.int64).cpu().numpy().reshape(1024, 4) / 1e3  # us
grid = nspec
st = st[:grid]
print("per CTA (us): spectrum mean %.0f  channel mean %.0f  wait mean %.0f  (min/max busy %.0f/%.0f)" % (
    st[:,0].mean(), st[:,1].mean(), st[:,2].mean(), (st[:,0]+st[:,1]).min(), (st[:,0]+st[:,1]).max()))
