"""Pins for oracle/cqplan.py against what the paper fixes (runs without a GPU).

Each test names the passage it pins.  None of them re-types the oracle's own
formula: they check worked numbers, closed forms and invariants.
"""
import math
import os

import numpy as np
import pytest

from oracle import cqplan
from synth.configs import CONFIGS, plan_args

GOLD = os.path.join(os.path.dirname(__file__), "golden", "table1_layout.txt")


def _golden(kind):
    rows = []
    for line in open(GOLD):
        if line.startswith("#") or not line.strip():
            continue
        f = line.split()
        if f[0] == kind:
            rows.append(f[1:])
    return rows


@pytest.mark.parametrize("row", _golden("layout"))
def test_table1_worked_examples(row):
    # SPEC S:123-125 / S:133 worked examples of Table 1
    fs, fmin, fmax, B, K, nch, xiK = row
    lay = cqplan.cq_layout(float(fs), float(fmin), float(fmax), int(B))
    assert lay.K == int(K)
    assert 2 * lay.K + 2 == int(nch)
    if xiK != "-":
        assert abs(lay.xi[-1] - float(xiK)) < 0.05
    # xi_max <= xi_K < fs/2
    assert lay.xi[-1] >= float(fmax) * (1 - 1e-12) and lay.xi[-1] < float(fs) / 2


@pytest.mark.parametrize("row", _golden("Q"))
def test_q_factor(row):
    B, q = row
    assert abs(cqplan.q_factor(int(B)) - float(q)) < 5e-7


def test_constant_q_bandwidth_identity():
    # Omega_k = xi_{k+1} - xi_{k-1} (k = 2..K-1) equals xi_k / Q (reading C3)
    lay = cqplan.cq_layout(44100.0, 50.0, 20000.0, 48)
    om_diff = lay.xi[2:] - lay.xi[:-2]
    assert np.max(np.abs(om_diff - lay.Omega[1:-1]) / lay.Omega[1:-1]) < 1e-12
    assert np.max(np.abs(lay.xi / lay.Omega - lay.Q)) < 1e-9 * lay.Q


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_config_plans_match_survey_table(cfg):
    row = [r for r in _golden("config") if int(r[0]) == cfg][0]
    _, K, lmin, lmax, l0, lk1, mmin, mmax, nM, sumM = map(int, row)
    p = cqplan.make_plan(*plan_args(CONFIGS[cfg]))
    Ls = [c.L for c in p.stored]
    assert p.layout.K == K
    assert (min(Ls[1:-1]), max(Ls[1:-1]), Ls[0], Ls[-1]) == (lmin, lmax, l0, lk1)
    M = p.M
    assert (M.min(), M.max(), len(set(M.tolist())), M.sum()) == (mmin, mmax, nM, sumM)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_plan_invariants(cfg):
    c = CONFIGS[cfg]
    p = cqplan.make_plan(*plan_args(c))
    Ls = p.sl_len
    K = p.layout.K
    # painless condition a_k <= L/L_k, i.e. M_k >= L_k (eq:framecond1), M_k even
    for ch in p.stored:
        assert ch.M >= ch.L and ch.M % 2 == 0 and cqplan.is_235_smooth(ch.M)
        assert ch.L >= 4  # C7 minimum width
    # Table 1 plateau widths: Omega_0 = 2 xi_min, Omega_{K+1} = fs - 2 xi_K,
    # in bins: support length ~ width * Ls/fs (integer rounding: +-1 bin)
    w0 = 2 * c.fmin * Ls / c.fs
    wN = (c.fs - 2 * p.layout.xi[-1]) * Ls / c.fs
    assert abs(p.stored[0].L - w0) <= 1.0 + 1e-9
    assert abs(p.stored[K + 1].L - wN) <= 1.0 + 1e-9
    # frame: the diagonal is positive everywhere (Prop. 2, eq:painlessframe1)
    assert p.D.min() > 0
    # union of supports covers the whole frequency axis
    cov = np.zeros(Ls, bool)
    for ch in p.full:
        cov[np.mod(ch.bins, Ls)] = True
    assert cov.all()
    # dual * D == g on every support (eq:painlessframe2)
    for ch, gd in zip(p.full, p.dual_full):
        np.testing.assert_allclose(gd * p.D[np.mod(ch.bins, Ls)], ch.g, rtol=1e-14, atol=1e-15)
    # the CQ filters peak at their centre bins omega_k = xi_k Ls/fs
    for k in (1, K // 2, K):
        ch = p.stored[k]
        om = p.layout.xi[k - 1] * Ls / c.fs
        assert abs(ch.bins[np.argmax(ch.g)] - om) <= 0.5 + 1e-9
    # mirror symmetry of the layout (Table 1 row K+2..2K+1): centres Ls - omega
    for kk in range(K + 2, 2 * K + 2):
        k = 2 * K + 2 - kk
        a, b = p.full[kk], p.stored[k]
        assert a.lo + a.L - 1 == Ls - b.lo and np.array_equal(a.g, b.g[::-1])


def test_frame_diagonal_symmetric_real_layout():
    # real signals: the filter layout is symmetric about Nyquist, so D[j] = D[Ls-j]
    p = cqplan.make_plan(*plan_args(CONFIGS[1]))
    Ls = p.sl_len
    j = np.arange(1, Ls)
    np.testing.assert_allclose(p.D[j], p.D[Ls - j], rtol=1e-14)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_partition_of_unity_and_dual_window(cfg):
    # eq:BUPU and dualwincond, <= 1e-12
    p = cqplan.make_plan(*plan_args(CONFIGS[cfg]))
    N = p.N
    pou = cqplan.periodize(p.h0, N)
    assert np.max(np.abs(pou - 1)) <= 1e-12
    dual = cqplan.periodize(p.h0 * p.h0dual, N)
    assert np.max(np.abs(dual - 1)) <= 1e-12
    # Tukey shape: essential length N, transitions tr, zero-padded to 2N
    t = np.arange(-N, N)
    assert np.all(p.h0[np.abs(t) <= (N - p.tr) // 2] == 1.0)
    assert np.all(p.h0[np.abs(t) >= (N + p.tr) // 2] == 0.0)
    assert np.count_nonzero(p.h0) == N + p.tr - 1
    # same support for the dual => at most 2 slices overlap each sample (C12)
    assert np.array_equal(p.h0 != 0, p.h0dual != 0)


def test_even_smooth_rounding():
    # C9: smallest even 2/3/5-smooth >= L
    assert [cqplan.smallest_even_smooth_ge(L) for L in (1, 3, 4, 7, 11, 13, 17, 49, 461, 906)] == \
        [2, 4, 4, 8, 12, 16, 18, 50, 480, 960]


@pytest.mark.parametrize("bad", [
    dict(fs=0.0), dict(fmin=-1.0), dict(fmin=30000.0), dict(fmax=10.0), dict(B=0),
    dict(sl_len=16386), dict(sl_len=7 * 1024), dict(tr=3), dict(tr=8192), dict(rasterize=3),
])
def test_invalid_parameters(bad):
    a = dict(fs=44100.0, fmin=65.4, fmax=22050.0, B=12, sl_len=16384, tr=2048, rasterize=0)
    a.update(bad)
    with pytest.raises(ValueError):
        cqplan.make_plan(a["fs"], a["fmin"], a["fmax"], a["B"], a["sl_len"], a["tr"], a["rasterize"])
