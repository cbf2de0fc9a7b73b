"""Per-hop kernel list of the real-time sliCQ (run under ncu --metrics gpu__time_duration.sum)."""
import sys
import numpy as np
import torch
from paper_1210_0084_b200 import api
from paper_1210_0084_b200.realtime import RealtimeSliCQ
from synth.configs import CONFIGS
from synth.signals import random_signal

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
graph = len(sys.argv) > 2 and sys.argv[2] == "graph"
plan = api.plan_for_config(CONFIGS[cfg])
rt = RealtimeSliCQ(plan, batch=1, graph=graph)
N = plan.N
x = random_signal(3, 1, 8 * N)
for k in range(8):
    rt.push(x[:, k * N:(k + 1) * N])
print("ok")
