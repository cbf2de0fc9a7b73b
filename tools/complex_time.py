"""Dev tool: complex-input sliCQ (slicq_forward_complex / slicq_inverse_complex) throughput on
cfg4's plan against the real path, CUDA events."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1210_0084_b200 import api
from synth.configs import CONFIGS
plan = api.plan_for_config(CONFIGS[4])
n = 1 << 26
x = (torch.randn(1, n, device="cuda") + 1j * torch.randn(1, n, device="cuda")).to(torch.complex64) * 0.1
xr = x.real.contiguous()
def t(fn, it=10):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it
c = plan.forward_complex(x); y = plan.inverse_complex(c, n)
cr = plan.forward(xr); yr = plan.inverse(cr, n)
tf, ti = t(lambda: plan.forward_complex(x, out=c)), t(lambda: plan.inverse_complex(c, n, out=y))
rf, ri = t(lambda: plan.forward(xr, out=cr)), t(lambda: plan.inverse(cr, n, out=yr))
err = ((y - x).abs().norm() / x.abs().norm()).item()
print(f"complex n=2^26: forward {tf:.3f} ms, inverse {ti:.3f} ms ({n / (tf + ti) / 1e6:.1f} G samples/s round trip), recon {err:.1e}")
print(f"real    n=2^26: forward {rf:.3f} ms, inverse {ri:.3f} ms (complex / real = {(tf + ti) / (rf + ri):.2f})")
