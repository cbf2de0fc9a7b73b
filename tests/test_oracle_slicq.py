"""Pins for oracle/slicq.py (Alg. 3/4) against the paper's propositions and identities."""
import numpy as np
import pytest

from oracle import cqplan, slicq
from synth.configs import CONFIGS, plan_args
from synth.signals import make_signal, random_signal


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("sl_len,tr,n", [(64, 8, 200), (96, 12, 96), (128, 16, 1000),
                                         (160, 4, 333), (256, 64, 2048), (512, 32, 1500)])
def test_sliced_perfect_reconstruction_small(sl_len, tr, n):
    # Prop. 3 with the canonical dual slicing window (C12): <= 1e-10
    p = cqplan.make_plan(8000.0, 150.0, None, 6, sl_len, tr, 0)
    x = random_signal(100 + sl_len, 2, n)
    c = slicq.forward(x, p)
    assert c.shape == (2, slicq.num_slices(n, sl_len), p.coeffs_per_slice)
    y = slicq.inverse(c, p, n)
    for b in range(2):
        assert _rel(y[b], x[b].astype(np.float64)) <= 1e-10


@pytest.mark.parametrize("raster", [0, 1, 2])
def test_sliced_perfect_reconstruction_cfg1(raster):
    # cfg1 parameters (BASELINE configs[0]) with every rasterization mode (C10)
    c1 = CONFIGS[1]
    p = cqplan.make_plan(c1.fs, c1.fmin, c1.fmax, c1.bins_per_octave, c1.sl_len, c1.tr_area, raster)
    x = make_signal(1)
    c = slicq.forward(x, p)
    y = slicq.inverse(c, p, x.shape[1])
    assert _rel(y[0], x[0].astype(np.float64)) <= 1e-10


def test_sinusoid_peaks_in_expected_channel():
    # constant-Q construction: a tone at f0 puts its energy in the CQ channel
    # whose centre is nearest f0 (north_star); cfg1 tones 220/1000/5000 Hz -> k = 22/48/76
    c1 = CONFIGS[1]
    p = cqplan.make_plan(*plan_args(c1))
    t = np.arange(c1.n) / c1.fs
    off = slicq.offsets(p)
    K = p.layout.K
    for f0, k_exp in ((220.0, 22), (1000.0, 48), (5000.0, 76)):
        x = (0.5 * np.sin(2 * np.pi * f0 * t)).astype(np.float32)[None]
        c = slicq.forward(x, p)[0]
        e = np.array([np.sum(np.abs(c[:, off[k]:off[k + 1]]) ** 2) for k in range(K + 2)])
        assert int(np.argmax(e[1:K + 1])) + 1 == k_exp
    # in the cfg1 mix each tone is a local maximum of the channel energy
    c = slicq.forward(make_signal(1), p)[0]
    e = np.array([np.sum(np.abs(c[:, off[k]:off[k + 1]]) ** 2) for k in range(K + 2)])
    for k in (22, 48, 76):
        assert e[k] > e[k - 1] and e[k] > e[k + 1]


def test_two_layer_bookkeeping():
    # P:320-323 and the identity of P:657-658:
    # s^0 + s^1 at n = m M_k/2 + n^s equals c^m[n^s + M_k/2] + c^{m+1}[n^s]; layers disjoint/complete
    p = cqplan.make_plan(8000.0, 150.0, None, 6, 128, 16, 0)
    n = 1000
    x = random_signal(4, 1, n)
    L = slicq.padded_length(n, 128)
    c = slicq.forward(x, p)[0]
    s = slicq.two_layer(c, p, L)
    S = c.shape[0]
    off = slicq.offsets(p)
    for k, ch in enumerate(p.stored):
        assert not np.isnan(s[k]).any()  # complete: every entry of both layers written once
        M, W = ch.M, s[k].shape[1]
        for m in range(S):
            for ns in range(M // 2):
                pos = (m * M // 2 + ns) % W
                lhs = s[k][0, pos] + s[k][1, pos]
                rhs = c[m, off[k] + ns + M // 2] + c[(m + 1) % S, off[k] + ns]
                assert lhs == rhs
    np.testing.assert_array_equal(slicq.from_two_layer(s, p, L), c)


def test_locality_linearity_zero():
    # S:179/S:203/S:266: zero in -> zero out; linear; an impulse where the window of slice m
    # vanishes gives exactly zero coefficients in slice m
    p = cqplan.make_plan(8000.0, 150.0, None, 6, 128, 16, 0)
    n = 640
    z = slicq.forward(np.zeros((1, n), np.float32), p)
    assert np.all(z == 0)
    a, b = random_signal(1, 1, n), random_signal(2, 1, n)
    ca, cb = slicq.forward(a, p), slicq.forward(b, p)
    cab = slicq.forward(a.astype(np.float64) + 3 * b.astype(np.float64), p)
    assert np.max(np.abs(cab - (ca + 3 * cb))) <= 1e-12 * np.max(np.abs(cab))
    N = p.N
    pos = 5 * N  # centre of slice 5: only slice 5 sees it (tr < N)
    x = np.zeros((1, n), np.float32)
    x[0, pos] = 1.0
    c = slicq.forward(x, p)[0]
    for m in range(c.shape[0]):
        if m != 5:
            assert np.all(c[m] == 0)
    assert np.any(c[5] != 0)


def test_inverse_samples_matches_full_inverse():
    p = cqplan.make_plan(8000.0, 150.0, None, 6, 128, 16, 0)
    n = 900
    x = random_signal(8, 1, n)
    c = slicq.forward(x, p)[0]
    y = slicq.inverse(c, p, n)[0]
    c_of = {m: c[m] for m in range(c.shape[0])}
    for a, b in ((0, 50), (130, 400), (850, 900)):
        np.testing.assert_allclose(slicq.inverse_samples(c_of, p, n, a, b), y[a:b], atol=1e-12)


@pytest.mark.parametrize("G", [2, 3, 5])
def test_sharded_emulation_equals_unsharded(G):
    # contiguous slice ranges, left halo of (N+tr)/2 samples with circular
    # wrap for rank 0, inverse spill added by the left neighbour
    p = cqplan.make_plan(8000.0, 150.0, None, 6, 128, 16, 0)
    n = 1234
    x = random_signal(21, 1, n)[0].astype(np.float64)
    N = p.N
    L = slicq.padded_length(n, p.sl_len)
    S = 2 * L // p.sl_len
    xp = np.zeros(L)
    xp[:n] = x
    halo = (N + p.tr) // 2
    c_ref = slicq.forward(x[None], p)[0]
    y_ref = slicq.inverse(c_ref[None], p, n)[0]
    bounds = [r * S // G for r in range(G + 1)]
    ys, spills = [], []
    for r in range(G):
        s0, s1 = bounds[r], bounds[r + 1]
        idx = np.mod(np.arange(s0 * N - halo, s1 * N), L)
        c_loc = slicq.forward_range(xp[idx], halo, s0, s1 - s0, p)
        np.testing.assert_allclose(c_loc, c_ref[s0:s1], rtol=0, atol=1e-11)
        y_loc, spill = slicq.inverse_range(c_ref[s0:s1], s0, s1 - s0, p, halo)
        ys.append(y_loc)
        spills.append(spill)
    for r in range(G):  # rank r receives rank r+1's spill (circularly)
        ys[r][-halo:] += spills[(r + 1) % G]
    y = np.concatenate(ys)[:n]
    np.testing.assert_allclose(y, y_ref, rtol=0, atol=1e-12)
