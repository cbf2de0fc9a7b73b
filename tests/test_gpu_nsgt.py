"""Full-length CQ-NSGT: slicq_nsgt_forward / slicq_nsgt_inverse against
the oracle's Alg. 1 (oracle.nsgt.analysis_real on the whole zero-padded signal) and perfect
reconstruction (Prop. 1), for L from 4096 to 2^17 (single-CTA and four-step spectrum paths)."""
import numpy as np
import pytest
import torch

from oracle import cqplan
from oracle import nsgt as onsgt
from synth.signals import random_signal

pytestmark = pytest.mark.gpu
TOL = 1e-5


@pytest.mark.parametrize("L,n,B,bpo,fmin,raster", [
    (4096, 4096, 2, 24, 50.0, 0), (16384, 12345, 1, 24, 50.0, 0), (32768, 32768, 1, 24, 50.0, 1),
    (65536, 65536, 1, 48, 50.0, 0), (131072, 100000, 2, 96, 60.0, 0)])
def test_nsgt_matches_oracle_and_reconstructs(L, n, B, bpo, fmin, raster):
    from paper_1210_0084_b200 import api
    # (M_k <= 1024 at every length: the channel-kernel limit)
    args = (44100.0, fmin, 22050.0, bpo, L, 64, raster)
    plan = api.Plan(*args)
    ref = cqplan.make_plan(*args)
    x = random_signal(L + n, B, n)
    xt = torch.from_numpy(x).cuda()
    c = plan.nsgt_forward(xt)
    y = plan.nsgt_inverse(c, n)
    torch.cuda.synchronize()
    cg = c.cpu().numpy().astype(np.complex128)
    for b in range(B):
        xp = np.zeros(L)
        xp[:n] = x[b]
        cr = np.concatenate(onsgt.analysis_real(xp, ref))
        err = np.linalg.norm(cg[b] - cr) / np.linalg.norm(cr)
        assert err <= TOL, (b, err)
        ry = np.linalg.norm(y[b].cpu().numpy() - x[b]) / np.linalg.norm(x[b])
        assert ry <= TOL, (b, ry)


def test_nsgt_rejects_long_input():
    from paper_1210_0084_b200 import api
    plan = api.Plan(44100.0, 50.0, 22050.0, 24, 4096, 64, 0)
    with pytest.raises(Exception):
        plan.nsgt_forward(torch.zeros(1, 4097, device="cuda"))
