"""The multi-GPU slice-range shard (dist.SliceRangeShard) on the library backend at world
size 1 (the halo is the circular wrap of the rank's own range): the side-stream
overlap of the boundary slice (halo exchange gated) with the interior gives exactly the
full transform's coefficients and output (bench.py --force-shard)."""
import pytest
import torch

from synth.signals import random_signal


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,batch", [(1, 1), (1, 2), (5, 1)])
def test_shard_world1_bit_identical_to_full(cfg, batch):
    from paper_1210_0084_b200 import api
    from paper_1210_0084_b200.dist import LibBackend, SliceRangeShard
    from synth.configs import CONFIGS
    plan = api.plan_for_config(CONFIGS[cfg])
    n = 9 * plan.N + 321
    x = torch.from_numpy(random_signal(8 + cfg, batch, n)).cuda()
    sh = SliceRangeShard(LibBackend(plan), n, batch=batch, rank=0, world=1)
    xl = sh.local_input(x)
    c = sh.forward(xl)
    y = sh.inverse(c)
    torch.cuda.synchronize()
    c_ref = plan.forward(x)
    y_ref = plan.inverse(c_ref, n)
    assert torch.equal(c, c_ref)
    assert torch.equal(y[:, :n], y_ref)
