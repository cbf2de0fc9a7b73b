"""Coefficient-domain helpers on host-only plans (index arithmetic, no kernels):
api.two_layer / api.from_two_layer (the paper's two-layer array s) against
the oracle's index-by-index construction (oracle.slicq.two_layer), and api.transpose_bins
 relocation / energy invariants (its audible effect, T8, is a GPU test in
tests/test_gpu_apps.py)."""
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


def test_transpose_bins_relocates_magnitudes():
    from paper_1210_0084_b200 import api
    plan = api.Plan(44100.0, 55.0, 22050.0, 24, 16384, 2048, 2, host_only=True)
    Ms, offs = plan.channel_lengths(), plan.channel_offsets()
    K = len(Ms) - 2
    M = int(Ms[1])
    rng = np.random.default_rng(3)
    S, C = 4, plan.coeffs_per_slice
    c = torch.from_numpy(rng.standard_normal((1, S, C)) + 1j * rng.standard_normal((1, S, C)))
    for s in (8, -8, 24):
        t = api.transpose_bins(plan, c, s)
        for k in range(1, K + 1):
            src = k - s
            blk = t[0, :, offs[k]:offs[k] + M]
            if 1 <= src <= K:  # magnitudes move verbatim (modulation only changes phase)
                assert torch.allclose(blk.abs(), c[0, :, offs[src]:offs[src] + M].abs(),
                                      rtol=1e-12, atol=0)
            else:
                assert torch.count_nonzero(blk) == 0
        # plateaus untouched; energy of the moved range preserved
        assert torch.equal(t[..., :offs[1]], c[..., :offs[1]])
        assert torch.equal(t[..., offs[K + 1]:], c[..., offs[K + 1]:])
        lo_src, hi_src = (1, K - s) if s > 0 else (1 - s, K)
        e_src = (c[..., offs[lo_src]:offs[hi_src + 1]].abs() ** 2).sum()
        e_dst = (t[..., offs[1]:offs[K + 1]].abs() ** 2).sum()
        assert abs(e_src - e_dst) <= 1e-12 * e_src
    with pytest.raises(ValueError):
        api.transpose_bins(api.Plan(44100.0, 55.0, 22050.0, 24, 16384, 2048, 0, host_only=True),
                           c[..., :1], 1)


def test_apply_mask_db_convention():
    """mask 0 -> 10^-5 (-100 dB), 1 -> 1 (0 dB), linear in dB in between."""
    from paper_1210_0084_b200 import api
    c = torch.full((1, 2, 6), 2.0 + 1.0j, dtype=torch.complex128)
    assert torch.equal(api.apply_mask(c, 1.0), c)
    assert torch.allclose(api.apply_mask(c, 0.0), c * 1e-5, rtol=1e-14, atol=0)
    m = torch.tensor([0.0, 0.25, 0.5, 0.75, 1.0, 0.5], dtype=torch.float64)
    out = api.apply_mask(c, m)
    want = 10.0 ** (-5.0 * (1.0 - m))
    assert torch.allclose(out[0, 1].abs() / c[0, 1].abs(), want, rtol=1e-12, atol=0)
    assert torch.allclose(20 * torch.log10(out[0, 0].abs() / c[0, 0].abs()), -100 * (1 - m))
    assert torch.equal(api.apply_mask(c, m, db=False), c * m)


def test_spectrogram_is_two_layer_sum():
    from paper_1210_0084_b200 import api
    plan = api.Plan(*plan_args(CONFIGS[1]), host_only=True)
    rng = np.random.default_rng(11)
    S, C = 8, plan.coeffs_per_slice
    c = torch.from_numpy(rng.standard_normal((1, S, C)) + 1j * rng.standard_normal((1, S, C)))
    sp = api.spectrogram(plan, c)
    s = api.two_layer(plan, c)
    for k in (0, 7, plan.num_channels - 1):
        assert torch.allclose(sp[k], (s[k][:, 0] + s[k][:, 1]).abs() ** 2)
        assert sp[k].shape[1] == S * int(plan.channel_lengths()[k]) // 2
