"""Sec. V-A / Fig. CoeffQual on the GPU: SNR of the sliCQ's
s^0 + s^1 against the full-length CQ-NSGT of the sampled system (Prop. 4), versus the
minimal filter width, for slice lengths 4096 / 16384 / 65536 and transition areas of 1/4
and 1/128 of the slice; Blackman-Harris filters.  Set-1-like inputs: seeded random signals
of 2^20 samples, complex like the paper's Set 1 (all 2K+2 channels) or, with --real, real
(stored channels); Set 2 (music) is not available.  Prints one JSON line per configuration
and a table."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1210_0084_b200 import api
from synth.signals import random_signal

L, BATCH = 2 ** 20, 8
BASE = (44100.0, 50.0, 22050.0, 48)
REAL = "--real" in sys.argv
xr = random_signal(2024, BATCH, L)
x = torch.from_numpy(xr if REAL else (xr + 1j * random_signal(2025, BATCH, L)).astype("complex64")).cuda()
rows = []
for N2 in (4096, 16384, 65536):
    for frac in (4, 128):
        tr = N2 // frac
        for mw in (2, 4, 6, 8, 12, 16, 24, 32):
            ps = api.Plan(*BASE, N2, tr, 0, window="blackman_harris", min_width=mw)
            pl = api.Plan(*BASE, L, tr, 0, window="blackman_harris", min_width=mw, sampled_from=N2)
            snr, _ = api.approximation_error(x, ps, pl)
            r = dict(input="real" if REAL else "complex", slice=N2, tr=f"1/{frac}", min_width=mw,
                     snr_db_mean=round(snr.mean().item(), 2),
                     snr_db_std=round(snr.std().item(), 3))
            rows.append(r)
            print(json.dumps(r), flush=True)
            ps.close(); pl.close()
print("| slice | tr | " + " | ".join(f"w={mw}" for mw in (2, 4, 6, 8, 12, 16, 24, 32)) + " |")
print("|---|---|" + "---|" * 8)
for N2 in (4096, 16384, 65536):
    for frac in (4, 128):
        v = [r["snr_db_mean"] for r in rows if r["slice"] == N2 and r["tr"] == f"1/{frac}"]
        print(f"| {N2} | 1/{frac} | " + " | ".join(f"{a:.1f}" for a in v) + " |")
