"""Dev probe: pinned host<->device copy bandwidth, alone and concurrent (e2e ceiling)."""
import torch, time
nb = 691200000
h_in = torch.empty(nb // 4, dtype=torch.float32, pin_memory=True)
h_out = torch.empty(nb // 4, dtype=torch.float32, pin_memory=True)
d_in = torch.empty(nb // 4, dtype=torch.float32, device="cuda")
d_out = torch.empty(nb // 4, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, it=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it
def h2d(): d_in.copy_(h_in, non_blocking=True)
def d2h(): h_out.copy_(d_out, non_blocking=True)
def both():
    cur = torch.cuda.current_stream(); s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    ms = t(fn)
    print(f"{name}: {ms:.2f} ms  {nb/ms/1e6:.1f} GB/s per direction")
