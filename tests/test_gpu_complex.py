"""Complex-input sliCQ on the GPU (slicq_forward_complex / slicq_inverse_complex, all 2K+2
channels) against the oracle's forward_complex / inverse_complex (tests/test_oracle_complex.py
pins it): per-slice coefficient relative L2 <= 1e-5 (C17) including the mirror channels,
reconstruction <= 1e-5, synthesis of arbitrary complex coefficients, and the real special
case equal to the real path."""
import numpy as np
import pytest
import torch

from oracle import cqplan
from oracle import slicq as osl
from synth.configs import CONFIGS, plan_args
from synth.signals import random_signal

pytestmark = pytest.mark.gpu
TOL = 1e-5


def _cx(seed, B, n):
    return (random_signal(seed, B, n) + 1j * random_signal(seed + 1000, B, n)).astype(np.complex64)


def _slice_err(cg, cr):
    rms = np.sqrt(np.mean(np.abs(cr) ** 2))
    return max(np.linalg.norm(cg[m] - cr[m]) / max(np.linalg.norm(cr[m]), rms * np.sqrt(cr.shape[1]))
               for m in range(cr.shape[0]))


@pytest.mark.parametrize("args,n,B", [
    ((8000.0, 150.0, 4000.0, 6, 4096, 512, 0), 3 * 4096 + 101, 2),
    ((44100.0, 65.4, 22050.0, 12, 16384, 2048, 1), 2 * 16384, 1),
    ((44100.0, 50.0, 22050.0, 48, 65536, 8192, 0), 65536 + 3, 1)])
def test_complex_matches_oracle_and_reconstructs(args, n, B):
    from paper_1210_0084_b200 import api
    plan = api.Plan(*args)
    ref = cqplan.make_plan(*args)
    assert plan.coeffs_per_slice_full == int(osl.offsets_full(ref)[-1])
    x = _cx(n, B, n)
    xt = torch.from_numpy(x).cuda()
    c = plan.forward_complex(xt)
    y = plan.inverse_complex(c, n)
    torch.cuda.synchronize()
    cr = osl.forward_complex(x.astype(np.complex128), ref)
    cg = c.cpu().numpy().astype(np.complex128)
    for b in range(B):
        assert _slice_err(cg[b], cr[b]) <= TOL
        ry = np.linalg.norm(y[b].cpu().numpy() - x[b]) / np.linalg.norm(x[b])
        assert ry <= TOL, ry


def test_complex_synthesis_of_arbitrary_coefficients():
    from paper_1210_0084_b200 import api
    args = (8000.0, 150.0, 4000.0, 6, 4096, 512, 0)
    plan = api.Plan(*args)
    ref = cqplan.make_plan(*args)
    n = 2 * 4096
    S = plan.num_slices(n)
    rng = np.random.default_rng(9)
    c = (rng.standard_normal((1, S, plan.coeffs_per_slice_full)) +
         1j * rng.standard_normal((1, S, plan.coeffs_per_slice_full))).astype(np.complex64)
    y = plan.inverse_complex(torch.from_numpy(c).cuda(), n).cpu().numpy()
    yr = osl.inverse_complex(c.astype(np.complex128), ref, n)
    assert np.linalg.norm(y - yr) / np.linalg.norm(yr) <= TOL


def test_complex_path_on_real_input_equals_real_path():
    from paper_1210_0084_b200 import api
    plan = api.plan_for_config(CONFIGS[1])
    n = 3 * plan.sl_len
    x = torch.from_numpy(random_signal(5, 1, n)).cuda()
    c = plan.forward_complex(x.to(torch.complex64))
    cs = plan.forward(x)
    C = plan.coeffs_per_slice
    torch.cuda.synchronize()
    assert torch.equal(c[:, :, :C], cs)  # same kernels on the real row; imaginary row is zero
