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


@pytest.mark.parametrize("L,n,B,bpo,fmin", [
    (2 ** 18, 2 ** 18, 2, 48, 50.0), (2 ** 19, 400000, 1, 24, 50.0),
    (2 ** 20, 2 ** 20, 2, 48, 50.0), (2 ** 21, 2 ** 21 - 1000, 1, 96, 60.0),
    (2 ** 22, 2 ** 22, 1, 96, 60.0), (2 ** 22, 3000000, 1, 48, 60.0)])
def test_long_nsgt_matches_oracle_and_reconstructs(L, n, B, bpo, fmin):
    """Long signals (kernels_long.cuh): four-step FFT_L with N1 = 512 .. 8192 columns,
    shared-memory mixed-radix channel FFTs (M_k <= 26000) and, at L = 2^22, the four-step
    channel FFTs through the staging scratch (M_k = 30720 = 2 x 15360, 60750 = 3 x 20250)."""
    from paper_1210_0084_b200 import api
    args = (44100.0, fmin, 22050.0, bpo, L, 64, 0)
    plan = api.Plan(*args)
    ref = cqplan.make_plan(*args)
    assert list(plan.channel_lengths()) == list(ref.M)
    x = random_signal(L + n + 7, B, n)
    xt = torch.from_numpy(x).cuda()
    c = plan.nsgt_forward(xt)
    y = plan.nsgt_inverse(c, n)
    torch.cuda.synchronize()
    cg = c.cpu().numpy().astype(np.complex128)
    for b in range(B):
        xp = np.zeros(L)
        xp[:n] = x[b]
        cr = onsgt.analysis_real(xp, ref)
        crc = np.concatenate(cr)
        err = np.linalg.norm(cg[b] - crc) / np.linalg.norm(crc)
        assert err <= TOL, (b, err)
        # per channel too (the small channels must not hide behind the big ones' energy)
        off = np.cumsum([0] + [len(v) for v in cr])
        rms = np.sqrt(np.mean(np.abs(crc) ** 2))
        for k, v in enumerate(cr):
            d = np.linalg.norm(cg[b, off[k]:off[k + 1]] - v) / max(np.linalg.norm(v), rms * np.sqrt(len(v)))
            assert d <= TOL, (b, k, d)
        ry = np.linalg.norm(y[b].cpu().numpy() - x[b]) / np.linalg.norm(x[b])
        assert ry <= TOL, (b, ry)


def test_long_plan_serves_only_the_full_length_transform():
    from paper_1210_0084_b200 import api
    plan = api.Plan(44100.0, 50.0, 22050.0, 48, 2 ** 18, 64, 0)
    with pytest.raises(Exception, match="full-length"):
        plan.forward(torch.zeros(1, 2 ** 18, device="cuda"))


def test_nsgt_rejects_long_input():
    from paper_1210_0084_b200 import api
    plan = api.Plan(44100.0, 50.0, 22050.0, 24, 4096, 64, 0)
    with pytest.raises(Exception):
        plan.nsgt_forward(torch.zeros(1, 4097, device="cuda"))


def test_long_nsgt_chunked_is_bit_identical(monkeypatch):
    """Long mode runs rows chunk by chunk when the staging budget is small (SLICQ_STAGE_MB,
    read at plan creation): identical coefficients and reconstruction."""
    from paper_1210_0084_b200 import api
    args = (44100.0, 50.0, 22050.0, 48, 2 ** 18, 64, 0)
    x = torch.from_numpy(random_signal(5, 5, 2 ** 18 - 3)).cuda()
    plan = api.Plan(*args)
    c = plan.nsgt_forward(x)
    y = plan.nsgt_inverse(c, x.shape[1])
    monkeypatch.setenv("SLICQ_STAGE_MB", "8")  # < 2 rows of staging per chunk
    small = api.Plan(*args)
    monkeypatch.delenv("SLICQ_STAGE_MB")
    assert small.kernel_launches("forward", 1, 5) > plan.kernel_launches("forward", 1, 5)
    c2 = small.nsgt_forward(x)
    y2 = small.nsgt_inverse(c2, x.shape[1])
    torch.cuda.synchronize()
    assert torch.equal(c, c2)
    assert torch.equal(y, y2)
