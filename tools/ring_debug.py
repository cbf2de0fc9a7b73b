"""Dev tool: locate ring-kernel disagreements (per channel / per unit) against the split path."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1210_0084_b200 import api
args = [float(v) if "." in v else int(v) for v in sys.argv[1].split(",")]
n = int(sys.argv[2]); env = sys.argv[3] if len(sys.argv) > 3 else ""
torch.manual_seed(0)
x = torch.randn(1, n, device="cuda") * 0.1
os.environ["SLICQ_FUSED"] = "0"
p0 = api.Plan(*args)
os.environ.pop("SLICQ_FUSED")
for kv in filter(None, env.split(",")):
    k, v = kv.split("="); os.environ[k] = v
p1 = api.Plan(*args)
c0 = p0.forward(x); c1 = p1.forward(x); torch.cuda.synchronize()
off = p0.channel_offsets(); M = p0.channel_lengths()
err = (c1 - c0).abs()[0]  # [S, C]
ref = c0.abs()[0].amax()
S = err.shape[0]
bad = []
for k in range(len(M)):
    e = err[:, off[k]:off[k + 1]].amax(dim=1)
    if e.max().item() > 1e-4 * ref.item():
        bad.append((k, int(M[k]), [int(s) for s in torch.nonzero(e > 1e-4 * ref).flatten()[:8]]))
print("units", S, "channels", len(M), "bad channels", len(bad))
for b in bad[:40]:
    print(b)
