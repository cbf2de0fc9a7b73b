"""api.two_layer / api.from_two_layer (the paper's two-layer coefficient array s, P:289,
P:320-323) against the oracle's index-by-index construction (oracle.slicq.two_layer), on a
host-only plan (pure index arithmetic: no kernels involved)."""
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
