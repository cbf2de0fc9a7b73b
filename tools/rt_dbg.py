import torch, numpy as np
from paper_1210_0084_b200 import api
from paper_1210_0084_b200.realtime import RealtimeSliCQ
from paper_1210_0084_b200.stream import ForwardStream, InverseStream
from paper_1210_0084_b200.dist import LibBackend
from synth.configs import CONFIGS
from synth.signals import random_signal
plan = api.plan_for_config(CONFIGS[1]); N=plan.N
H=6
x = torch.from_numpy(random_signal(77, 1, H*N))
for graph in (False, True):
    rt = RealtimeSliCQ(plan, batch=1, graph=graph)
    h=rt.halo
    ys=[rt.push(x[:, k*N:(k+1)*N]) for k in range(H)]
    y=torch.cat(ys,1)
    for k in range(H):
        seg = y[:, k*N:(k+1)*N]; ref = torch.zeros_like(seg)
        lo = k*N-h
        a=max(lo,0); ref[:, a-lo:] = x[:, a:lo+N]
        print(graph, k, float((seg-ref).norm()/ref.norm().clamp_min(1e-9)), float(seg.norm()))
be=LibBackend(plan); xd=x.cuda()
fs,inv=ForwardStream(be,batch=1,device=xd.device),InverseStream(be,batch=1)
ys=[inv.push(fs.push(xd[:, k*N:(k+1)*N])) for k in range(H)]
y=torch.cat([t for t in ys if t is not None],1).cpu()
print("stream err", float((y-x[:, :y.shape[1]]).norm()/x[:, :y.shape[1]].norm()), y.shape)
