"""Dev tool: TMA-staged vs global-load channel kernels (SLICQ_TB) -- where do they differ?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1210_0084_b200 import api
from synth.configs import CONFIGS
from synth.signals import random_signal
cfg = int(sys.argv[1]); n = int(sys.argv[2]); batch = int(sys.argv[3])
x = torch.from_numpy(random_signal(4242 + cfg, batch, n)).cuda()
os.environ["SLICQ_TB"] = "0"; p0 = api.plan_for_config(CONFIGS[cfg])
os.environ["SLICQ_TB"] = "1"; p1 = api.plan_for_config(CONFIGS[cfg])
c0, c1 = p0.forward(x), p1.forward(x); torch.cuda.synchronize()
d = (c0 - c1).abs()
print("fwd equal", torch.equal(c0, c1), "max diff", d.max().item(), "max |c|", c0.abs().max().item())
off = np.asarray(p0.channel_offsets() if hasattr(p0, "channel_offsets") else [])
dd = d.reshape(-1, d.shape[-1]).amax(0).cpu().numpy()
bad = np.nonzero(dd > 1e-6 * c0.abs().max().item())[0]
print("bad columns", len(bad), bad[:20], bad[-5:] if len(bad) else "")
if len(off):
    ks = sorted(set(np.searchsorted(off, bad, side="right") - 1))
    print("bad channels", ks[:40], "of", len(off) - 1)
ds = d.reshape(-1, d.shape[-1]).amax(1).cpu().numpy()
print("bad units", np.nonzero(ds > 1e-6 * c0.abs().max().item())[0][:40], "of", ds.size)
y0, y1 = p0.inverse(c0, n), p1.inverse(c0, n); torch.cuda.synchronize()
print("inv equal", torch.equal(y0, y1), "max diff", (y0 - y1).abs().max().item())
