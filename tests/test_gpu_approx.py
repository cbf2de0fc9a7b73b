"""Prop. 4 / Sec. V-A on the GPU: slicq_approx_error over the library's
sliCQ (slicq_forward) and full-length CQ-NSGT of the sampled system (slicq_nsgt_forward,
plan_create_ex2(sampled_from = 2N), long mode) against the oracle's sums and SNR
(oracle/approx.py, pinned by tests/test_oracle_approx.py)."""
import numpy as np
import pytest
import torch

from oracle import approx, cqplan
from oracle import nsgt as onsgt
from synth.signals import random_signal

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("window,mw,tr,B", [("blackman_harris", 4, 1024, 24),
                                            ("blackman_harris", 16, 32, 24),
                                            ("hann", 8, 1024, 12)])
def test_approx_error_matches_oracle(window, mw, tr, B):
    from paper_1210_0084_b200 import api
    N2, L = 4096, 2 ** 18
    base = (44100.0, 50.0, 22050.0, B)
    ps = api.Plan(*base, N2, tr, 0, window=window, min_width=mw)
    pl = api.Plan(*base, L, tr, 0, window=window, min_width=mw, sampled_from=N2)
    ops = cqplan.make_plan(*base, N2, tr, 0, window=window, min_width=mw)
    opl = cqplan.make_plan(*base, L, tr, 0, window=window, min_width=mw, sampled_from=N2)
    assert list(pl.channel_lengths()) == list(opl.M)
    x = random_signal(mw * 1000 + tr, 2, L)
    snr, sums = api.approximation_error(torch.from_numpy(x).cuda(), ps, pl)
    torch.cuda.synchronize()
    sums = sums.cpu().numpy()
    for b in range(2):
        ref = approx.channel_sums(x[b].astype(np.float64), ops, opl)
        np.testing.assert_allclose(sums[b, :, 0], ref[:, 0], rtol=1e-5)
        # the error energy is a difference of close coefficient sets: compare in dB
        err_db = 10 * np.log10(sums[b, :, 1].sum() / ref[:, 1].sum())
        assert abs(err_db) < 0.05, err_db
        ref_snr = 10 * np.log10(ref[:, 0].sum() / ref[:, 1].sum())
        assert abs(snr[b].item() - ref_snr) < 0.05, (snr[b].item(), ref_snr)


def test_sampled_system_analysis_and_refusals():
    """The full-length analysis of a non-painless sampled system folds aliased bins
    (Alg. 1 periodisation) -- checked against the oracle; synthesis is refused."""
    from paper_1210_0084_b200 import api
    N2, L = 4096, 2 ** 18
    base = (44100.0, 50.0, 22050.0, 24)
    pl = api.Plan(*base, L, 1024, 0, window="blackman_harris", min_width=4, sampled_from=N2)
    opl = cqplan.make_plan(*base, L, 1024, 0, window="blackman_harris", min_width=4,
                           sampled_from=N2)
    assert not opl.painless
    x = random_signal(77, 1, L)
    c = pl.nsgt_forward(torch.from_numpy(x).cuda()).cpu().numpy()[0].astype(np.complex128)
    cr = np.concatenate(onsgt.analysis_real(x[0].astype(np.float64), opl))
    assert np.linalg.norm(c - cr) / np.linalg.norm(cr) <= 1e-5
    with pytest.raises(Exception, match="painless"):
        pl.nsgt_inverse(torch.from_numpy(c.astype(np.complex64)).cuda()[None], L)
    with pytest.raises(Exception):  # a non-painless system below the long path
        api.Plan(*base, 65536, 1024, 0, window="blackman_harris", min_width=4, sampled_from=N2)


def test_approx_error_complex_matches_oracle():
    """Complex Set-1-like signals over all 2K+2 channels (slicq_approx_error_complex)."""
    from paper_1210_0084_b200 import api
    N2, L = 4096, 2 ** 18
    base = (44100.0, 50.0, 22050.0, 24)
    ps = api.Plan(*base, N2, 1024, 0, window="blackman_harris", min_width=8)
    pl = api.Plan(*base, L, 1024, 0, window="blackman_harris", min_width=8, sampled_from=N2)
    ops = cqplan.make_plan(*base, N2, 1024, 0, window="blackman_harris", min_width=8)
    opl = cqplan.make_plan(*base, L, 1024, 0, window="blackman_harris", min_width=8,
                           sampled_from=N2)
    x = (random_signal(31, 1, L) + 1j * random_signal(32, 1, L)).astype(np.complex64)
    snr, sums = api.approximation_error(torch.from_numpy(x).cuda(), ps, pl)
    torch.cuda.synchronize()
    sums = sums.cpu().numpy()[0]
    ref = approx.channel_sums_complex(x[0].astype(np.complex128), ops, opl)
    assert sums.shape == ref.shape
    np.testing.assert_allclose(sums[:, 0], ref[:, 0], rtol=1e-5)
    ref_snr = 10 * np.log10(ref[:, 0].sum() / ref[:, 1].sum())
    assert abs(snr[0].item() - ref_snr) < 0.05, (snr[0].item(), ref_snr)


def test_nsgt_complex_roundtrip_and_oracle():
    from paper_1210_0084_b200 import api
    args = (44100.0, 50.0, 22050.0, 48, 2 ** 18, 64, 0)
    plan = api.Plan(*args)
    ref = cqplan.make_plan(*args)
    n = 2 ** 18 - 5
    x = (random_signal(41, 1, n) + 1j * random_signal(42, 1, n)).astype(np.complex64)
    xt = torch.from_numpy(x).cuda()
    c = plan.nsgt_forward_complex(xt)
    y = plan.nsgt_inverse_complex(c, n)
    torch.cuda.synchronize()
    xp = np.zeros(2 ** 18, np.complex128)
    xp[:n] = x[0]
    cr = np.concatenate(onsgt.analysis(xp, ref.full, 2 ** 18))
    cg = c.cpu().numpy()[0].astype(np.complex128)
    assert np.linalg.norm(cg - cr) / np.linalg.norm(cr) <= 1e-5
    assert np.linalg.norm(y.cpu().numpy()[0] - x[0]) / np.linalg.norm(x[0]) <= 1e-5
