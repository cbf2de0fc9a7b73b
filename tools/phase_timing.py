"""Per-phase cycle breakdown of the forward / inverse kernels (dev tool).

Uses libslicq_dbg.so (built with -DSLICQ_PHASE_TIMING): thread 0 of each CTA adds clock64
deltas between __syncthreads-separated phases.  Prints average cycles per CTA per phase."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SLICQ_LIB"] = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "paper_1210_0084_b200", "libslicq_dbg.so")
import torch
from paper_1210_0084_b200 import api, _lib
from synth.configs import CONFIGS
cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4 * 148 * 8192
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 1
plan = api.plan_for_config(cfg)
L = _lib.lib()
f = L.slicq_debug_phase_times
f.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
logN = (plan.N).bit_length() - 1
x = torch.randn(batch, n, device="cuda") * 0.1
c = plan.forward(x); y = plan.inverse(c, n); torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 32)()
f(logN, buf, 1)
plan.forward(x, out=c); plan.inverse(c, n, out=y); torch.cuda.synchronize()
f(logN, buf, 0)
nct = batch * c.shape[1]
names_f = ["pass1+load", "pass2", "pass3", "r2c pack", "channels"]
names_i = ["channels", "c2r pack", "pass1", "pass2", "pass3+epilogue", "pairing"]
tf = sum(buf[i] for i in range(5)); ti = sum(buf[16 + i] for i in range(6))
print(f"config {cfg.name}: {nct} CTAs; cycles per CTA (thread 0, incl. waits)")
for i, nm in enumerate(names_f):
    print(f"  fwd {nm:16s} {buf[i]/nct:10.0f}  {100*buf[i]/max(tf,1):5.1f}%")
for i, nm in enumerate(names_i):
    print(f"  inv {nm:16s} {buf[16+i]/nct:10.0f}  {100*buf[16+i]/max(ti,1):5.1f}%")
