"""Dev probe: does running two independent half-size calls on two streams beat one call?
(tests whether the spectrum and channel kernels fill each other's idle phases)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1210_0084_b200 import api
from synth.configs import CONFIGS
cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
n = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.n
parts = int(sys.argv[3]) if len(sys.argv) > 3 else 2
plans = [api.plan_for_config(cfg) for _ in range(parts)]
x = torch.randn(1, n, device="cuda") * 0.1
xs = [x[:, i * (n // parts):(i + 1) * (n // parts)].contiguous() for i in range(parts)]
streams = [torch.cuda.Stream() for _ in range(parts)]
cs = [p.forward(xi) for p, xi in zip(plans, xs)]
ys = [p.inverse(c, xi.shape[1]) for p, c, xi in zip(plans, cs, xs)]
torch.cuda.synchronize()

def timeit(fn, it=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it

def seq_fwd():
    for p, xi, c in zip(plans, xs, cs): p.forward(xi, out=c)
def par_fwd():
    cur = torch.cuda.current_stream()
    for s in streams: s.wait_stream(cur)
    for p, xi, c, s in zip(plans, xs, cs, streams): p.forward(xi, out=c, stream=s)
    for s in streams: cur.wait_stream(s)
def seq_inv():
    for p, c, y, xi in zip(plans, cs, ys, xs): p.inverse(c, xi.shape[1], out=y)
def par_inv():
    cur = torch.cuda.current_stream()
    for s in streams: s.wait_stream(cur)
    for p, c, y, xi, s in zip(plans, cs, ys, xs, streams): p.inverse(c, xi.shape[1], out=y, stream=s)
    for s in streams: cur.wait_stream(s)
print(f"parts={parts} seq fwd {timeit(seq_fwd):.3f} ms  par fwd {timeit(par_fwd):.3f} ms  "
      f"seq inv {timeit(seq_inv):.3f} ms  par inv {timeit(par_inv):.3f} ms", flush=True)
