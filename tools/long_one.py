import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_1210_0084_b200 import api
L, B = 2 ** 20, 16
plan = api.Plan(44100.0, 50.0, 22050.0, 48, L, 64, 0)
x = torch.randn(B, L, device="cuda") * 0.1
c = plan.nsgt_forward(x)
y = plan.nsgt_inverse(c, L)
torch.cuda.synchronize()
print("ok")
