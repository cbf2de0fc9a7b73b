"""Coefficient-domain operations: api.two_layer / api.from_two_layer (the paper's two-layer
array s; index views on host-only plans, no GPU) against the oracle's
index-by-index construction (oracle.slicq.two_layer), and the device kernels of NEXT-4
(`-m gpu`): slicq_transpose_bins, slicq_apply_mask and slicq_spectrogram
 against numpy references (their audible effects, T8 and the mask decomposition,
are in tests/test_gpu_apps.py)."""
import numpy as np
import pytest
import torch

from oracle import cqplan
from oracle import slicq as oslicq
from synth.configs import CONFIGS, plan_args


@pytest.mark.parametrize("cfg_id,S", [(1, 8), (2, 6)])
def test_two_layer_matches_oracle(cfg_id, S):
    from paper_1210_0084_b200 import api
    cfg = CONFIGS[cfg_id]
    plan = api.Plan(*plan_args(cfg), host_only=True)
    ref = cqplan.make_plan(*plan_args(cfg))
    C = plan.coeffs_per_slice
    rng = np.random.default_rng(cfg_id)
    c = rng.standard_normal((2, S, C)) + 1j * rng.standard_normal((2, S, C))
    ct = torch.from_numpy(c)
    s = api.two_layer(plan, ct)
    L = S * plan.N
    for b in range(2):
        so = oslicq.two_layer(c[b], ref, L)
        for k in range(plan.num_channels):
            assert np.array_equal(s[k][b].numpy(), so[k]), k
    back = api.from_two_layer(plan, s)
    assert torch.equal(back, ct)
    # s0 + s1 at n = m M/2 + n^s sums slice m's second half and slice m+1's first
    k = plan.num_channels // 2
    M = int(plan.channel_lengths()[k])
    off = int(plan.channel_offsets()[k])
    m, ns = 2, 1  # n^s < M/2
    tot = s[k][0, 0] + s[k][0, 1]  # batch row 0: s^0 + s^1
    want = c[0, m, off + ns + M // 2] + c[0, m + 1, off + ns]
    assert np.isclose(tot[m * M // 2 + ns].item(), want)


@pytest.mark.gpu
def test_transpose_bins_relocates_magnitudes():
    """slicq_transpose_bins: magnitudes move verbatim by the shift, the modulation
    is e^{2 pi i d n/M} with d the centre-bin difference, vacated channels are zero, the
    plateaus are copied; non-rasterised plans are refused."""
    from paper_1210_0084_b200 import api
    plan = api.Plan(44100.0, 55.0, 22050.0, 24, 16384, 2048, 2)
    ex = plan.export()
    Ms, offs = plan.channel_lengths(), plan.channel_offsets()
    K = len(Ms) - 2
    M = int(Ms[1])
    centre = ex["lo"].astype(np.float64) + (ex["len"].astype(np.float64) - 1.0) / 2.0
    rng = np.random.default_rng(3)
    S, C = 4, plan.coeffs_per_slice
    c = (rng.standard_normal((1, S, C)) + 1j * rng.standard_normal((1, S, C))).astype(np.complex64)
    ct = torch.from_numpy(c).cuda()
    n = np.arange(M)
    for s in (8, -8, 24):
        t = api.transpose_bins(plan, ct, s).cpu().numpy()
        for k in range(1, K + 1):
            src = k - s
            blk = t[0, :, offs[k]:offs[k] + M]
            if 1 <= src <= K:
                d = int(round(centre[k] - centre[src]))
                want = c[0, :, offs[src]:offs[src] + M] * np.exp(2j * np.pi * d * n / M)
                assert np.abs(blk - want).max() <= 1e-5 * np.abs(want).max()
            else:
                assert np.count_nonzero(blk) == 0
        assert np.array_equal(t[..., :offs[1]], c[..., :offs[1]])
        assert np.array_equal(t[..., offs[K + 1]:], c[..., offs[K + 1]:])
    with pytest.raises(Exception):
        api.transpose_bins(api.Plan(44100.0, 55.0, 22050.0, 24, 16384, 2048, 0),
                           torch.zeros((1, 2, C), dtype=torch.complex64, device="cuda"), 1)


@pytest.mark.gpu
def test_apply_mask_db_convention():
    """slicq_apply_mask: mask 0 -> 10^-5 (-100 dB), 1 -> 1 (0 dB), linear in dB in
    between; per-column and full-grid masks."""
    from paper_1210_0084_b200 import api
    plan = api.Plan(*plan_args(CONFIGS[1]))
    C = plan.coeffs_per_slice
    c = torch.full((2, 3, C), 2.0 + 1.0j, dtype=torch.complex64, device="cuda")
    assert torch.equal(api.apply_mask(plan, c, 1.0), c)
    assert torch.allclose(api.apply_mask(plan, c, 0.0), c * 1e-5, rtol=1e-6, atol=0)
    m = torch.rand(C, dtype=torch.float32, device="cuda")
    out = api.apply_mask(plan, c, m)
    want = 10.0 ** (-5.0 * (1.0 - m.double()))
    assert torch.allclose((out[1, 2].abs() / c[1, 2].abs()).double(), want, rtol=1e-5, atol=0)
    assert torch.allclose(20 * torch.log10((out[0, 0].abs() / c[0, 0].abs()).double()),
                          -100 * (1 - m.double()), atol=1e-3)
    g = torch.rand(c.shape, dtype=torch.float32, device="cuda")
    assert torch.equal(api.apply_mask(plan, c, g, db=False), c * g)
    c2 = c.clone()
    api.apply_mask(plan, c2, g, db=False, inplace=True)
    assert torch.equal(c2, c * g)


@pytest.mark.gpu
def test_spectrogram_is_two_layer_sum():
    """slicq_spectrogram = |s^0 + s^1|^2 of the two-layer array, per channel."""
    from paper_1210_0084_b200 import api
    plan = api.Plan(*plan_args(CONFIGS[1]))
    rng = np.random.default_rng(11)
    S, C = 8, plan.coeffs_per_slice
    c = (rng.standard_normal((2, S, C)) + 1j * rng.standard_normal((2, S, C))).astype(np.complex64)
    sp = api.spectrogram(plan, torch.from_numpy(c).cuda())
    ref = cqplan.make_plan(*plan_args(CONFIGS[1]))
    L = S * plan.N
    for b in range(2):
        so = oslicq.two_layer(c[b].astype(np.complex128), ref, L)
        for k in (0, 7, plan.num_channels - 1):
            want = np.abs(so[k][0] + so[k][1]) ** 2
            got = sp[k][b].cpu().numpy()
            assert got.shape == want.shape
            assert np.abs(got - want).max() <= 1e-5 * want.max()
