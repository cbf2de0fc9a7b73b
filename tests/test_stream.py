"""Streaming sliCQ (paper_1210_0084_b200/stream.py): a stream pushed in
arbitrary chunks gives exactly the coefficients of one slice-range call over the whole
zero-headed signal, and the streaming synthesis reconstructs it (Prop. 3).
CPU tests drive the stream logic with the oracle's range functions; the GPU tests run the
library's range kernels."""
import numpy as np
import pytest
import torch

from oracle import cqplan
from oracle import slicq as oslicq
from paper_1210_0084_b200.stream import ForwardStream, InverseStream
from synth.signals import random_signal

ARGS = (8000.0, 150.0, None, 6, 128, 16, 0)


class OracleBackend:
    """Range backend over the oracle's fp64 functions (CPU tensors)."""

    def __init__(self, args=ARGS):
        self.p = cqplan.make_plan(*args)
        self.N = self.p.N
        self.halo = (self.p.N + self.p.tr) // 2

    def forward_range(self, x_local, halo, slice0, nslices, total_slices):
        out = [oslicq.forward_range(x_local[b].numpy(), halo, slice0, nslices, self.p)
               for b in range(x_local.shape[0])]
        return torch.from_numpy(np.stack(out))

    def inverse_range(self, c_local, slice0, nslices, total_slices, halo):
        ys, sps = [], []
        for b in range(c_local.shape[0]):
            y, sp = oslicq.inverse_range(c_local[b].numpy(), slice0, nslices, self.p, halo)
            ys.append(y)
            sps.append(sp)
        return torch.from_numpy(np.stack(ys)), torch.from_numpy(np.stack(sps))

    def overlap_add(self, y_tail, spill):
        y_tail += spill


def _chunks(n, rng, lo=1, hi=300):
    out, pos = [], 0
    while pos < n:
        m = int(rng.integers(lo, hi))
        out.append((pos, min(n, pos + m)))
        pos += m
    return out


def _run_stream(backend, x, rng, dtype):
    fs = ForwardStream(backend, batch=x.shape[0], dtype=dtype, device=x.device)
    inv = InverseStream(backend, batch=x.shape[0])
    coeffs, ys = [], []
    for a, b in _chunks(x.shape[1], rng):
        c = fs.push(x[:, a:b])
        if c is not None:
            coeffs.append(c)
            ys.append(inv.push(c))
    c = fs.flush()
    if c is not None:
        coeffs.append(c)
        ys.append(inv.push(c))
    ys.append(inv.flush())
    return torch.cat(coeffs, dim=1), torch.cat(ys, dim=1)


def _zero_headed(x, halo, nsl, N):
    B, n = x.shape
    xl = torch.zeros((B, halo + nsl * N), dtype=x.dtype, device=x.device)
    xl[:, halo:halo + n] = x
    return xl


@pytest.mark.parametrize("n,batch,seed", [(1000, 1, 1), (2048, 2, 2), (130, 1, 3)])
def test_stream_oracle_matches_one_range_call(n, batch, seed):
    be = OracleBackend()
    x = torch.from_numpy(random_signal(seed, batch, n).astype(np.float64))
    c, y = _run_stream(be, x, np.random.default_rng(seed), torch.float64)
    N, halo = be.N, be.halo + (be.halo & 1)
    K = (n + be.halo - 1) // N + 1  # slices whose windows reach the signal
    assert c.shape[1] == K
    ref = be.forward_range(_zero_headed(x, halo, K, N), halo, 0, K, 1 << 40)
    assert torch.equal(c, ref)  # same slice computations, any chunking
    # synthesis: the whole stream is recovered (zero head, zero tail: PoU holds on [0, n))
    assert y.shape[1] >= n
    assert torch.allclose(y[:, :n], x, atol=1e-10, rtol=0)


def test_stream_oracle_head_differs_from_circular():
    """The streaming head is zero history, not the circular wrap of P:328: slice 0 of a
    stream sees zeros where the finite-signal transform sees the signal's tail."""
    be = OracleBackend()
    n = 4 * be.N
    x = torch.from_numpy(random_signal(7, 1, n).astype(np.float64))
    c, _ = _run_stream(be, x, np.random.default_rng(7), torch.float64)
    circ = oslicq.forward(x[0].numpy(), be.p)[0]  # [S][C]
    assert np.allclose(c[0, 1].numpy(), circ[1], atol=1e-12)  # interior slice identical
    assert not np.allclose(c[0, 0].numpy(), circ[0], atol=1e-6)  # head differs


@pytest.mark.gpu
def test_stream_gpu_matches_range_call_and_reconstructs():
    from paper_1210_0084_b200 import api
    from paper_1210_0084_b200.dist import LibBackend
    from synth.configs import CONFIGS
    plan = api.plan_for_config(CONFIGS[1])
    be = LibBackend(plan)
    n, batch = 5 * plan.N + 123, 2
    x = torch.from_numpy(random_signal(99, batch, n)).cuda()
    rng = np.random.default_rng(5)
    fs = ForwardStream(be, batch=batch, device=x.device)
    inv = InverseStream(be, batch=batch)
    coeffs, ys = [], []
    for a, b in _chunks(n, rng, 1000, 20000):
        c = fs.push(x[:, a:b])
        if c is not None:
            coeffs.append(c)
            ys.append(inv.push(c))
    c = fs.flush()
    if c is not None:
        coeffs.append(c)
        ys.append(inv.push(c))
    ys.append(inv.flush())
    c, y = torch.cat(coeffs, dim=1), torch.cat(ys, dim=1)
    torch.cuda.synchronize()
    N, halo = plan.N, plan.halo + (plan.halo & 1)
    K = (n + plan.halo - 1) // N + 1
    ref = plan.forward_range(_zero_headed(x, halo, K, N), halo, 0, K, 1 << 40)
    assert torch.equal(c, ref)
    err = ((y[:, :n] - x).norm() / x.norm()).item()
    assert err <= 1e-5, err
    # against the oracle's zero-headed range transform (C17 tolerance per slice)
    from synth.configs import plan_args
    op = cqplan.make_plan(*plan_args(CONFIGS[1]))
    xo = _zero_headed(x.cpu().double(), halo, K, N)[0].numpy()
    co = oslicq.forward_range(xo, halo, 0, K, op)
    cg = c[0].cpu().numpy()
    rms = np.sqrt(np.mean(np.abs(co) ** 2))
    for m in range(K):
        d = np.linalg.norm(cg[m] - co[m]) / max(np.linalg.norm(co[m]), rms * np.sqrt(co.shape[1]))
        assert d <= 1e-5, (m, d)
