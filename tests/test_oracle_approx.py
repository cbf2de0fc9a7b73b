"""Pins of the Prop. 4 / Sec. V-A oracle (oracle/approx.py, test T5) and
the host plan's filter options (plan_create_ex2) against it.

  * Blackman-Harris H: the 4-term window's defining values (reading C20)
  * the sampled system: g_k[j] = g^L_k[j L/2N] and M^L_k = (L/2N) M_k (C21)
  * the Prop. 4 normalisation: Alg. 1 coefficients / sqrt(L a_k) = <f, T_{n a_k} g-check>
    by direct inner products (C22)
  * the proof's identity s^0 + s^1 - c = R[n] (C24) by direct inner products --
    pins the sliCQ oracle, the two-layer array and the sampled system together
  * the bound eq:inner_outer
  * the trend of Fig. CoeffQual: SNR grows with the minimal filter width
"""
import numpy as np
import pytest

from oracle import approx, cqplan

FS = 8000.0
BASE = (FS, 200.0, None, 6)


def _pair(window, min_width, tr=32, N2=256, L=2048, raster=0):
    ps = cqplan.make_plan(*BASE, N2, tr, raster, window=window, min_width=min_width)
    pl = cqplan.make_plan(*BASE, L, tr, raster, window=window, min_width=min_width,
                          sampled_from=N2)
    return ps, pl


def test_blackman_harris_values():
    H = cqplan.blackman_harris
    assert H(np.array([0.0]))[0] == pytest.approx(1.0, abs=1e-15)        # a0+a1+a2+a3 = 1
    assert H(np.array([0.5]))[0] == pytest.approx(0.35875 - 0.48829 + 0.14128 - 0.01168, abs=1e-15)
    x = np.linspace(-0.5, 0.5, 101)
    assert np.allclose(H(x), H(-x), atol=1e-15)
    assert np.all(H(np.array([0.51, -0.7, 3.0])) == 0.0)
    assert np.all(np.diff(H(np.linspace(0, 0.5, 50))) < 0)                 # monotone lobe


@pytest.mark.parametrize("window,mw,raster", [("hann", 4, 0), ("blackman_harris", 8, 0),
                                              ("blackman_harris", 32, 1), ("hann", 16, 2)])
def test_sampled_system(window, mw, raster):
    ps, pl = _pair(window, mw, raster=raster)
    sc = pl.sl_len // ps.sl_len
    for a, b in zip(ps.stored, pl.stored):
        assert b.M == sc * a.M
        vals = dict(zip(b.bins.tolist(), b.g))
        for j, gv in zip(a.bins.tolist(), a.g):
            assert abs(vals.get(sc * j, 0.0) - gv) <= 1e-12
        # and no fine-grid multiple of sc outside the slice support carries a value
        mult = [j for j in b.bins.tolist() if j % sc == 0]
        assert sorted(j // sc for j in mult) == a.bins.tolist()


def test_p4_normalisation_is_the_inner_product():
    ps, pl = _pair("blackman_harris", 8)
    f = np.random.default_rng(3).standard_normal(pl.sl_len)
    c = approx.full_coeffs(f, pl)
    for k in (0, 3, len(pl.stored) - 1):
        ch = pl.stored[k]
        a = pl.sl_len / ch.M
        direct = np.array([np.vdot(approx.atom(ch, pl.sl_len, n * a), f) for n in range(ch.M)])
        assert np.abs(direct - c[k]).max() <= 1e-10 * np.abs(c[k]).max()


@pytest.mark.parametrize("window,mw,tr", [("blackman_harris", 8, 32), ("hann", 4, 96),
                                          ("blackman_harris", 24, 2)])
def test_prop4_identity_and_bound(window, mw, tr):
    ps, pl = _pair(window, mw, tr=tr)
    f = np.random.default_rng(11).standard_normal(pl.sl_len)
    c = approx.full_coeffs(f, pl)
    s = approx.slice_sum(f, ps, pl.sl_len)
    for k in range(len(pl.stored)):
        R, bound = approx.residual_and_bound(f, ps, pl, k)
        scale = np.abs(c[k]).max()
        assert np.abs((s[k] - c[k]) - R).max() <= 1e-10 * scale, k
        assert np.all(np.abs(R) <= bound * (1 + 1e-12)), k


def test_prop4_identity_single_slice_pair():
    """L = 2N: no circular overspill (the sum over j in eq:inner_outer is empty)."""
    ps, pl = _pair("hann", 8, N2=512, L=512)
    f = np.random.default_rng(5).standard_normal(512)
    c = approx.full_coeffs(f, pl)
    s = approx.slice_sum(f, ps, 512)
    for k in (1, 5):
        R, _ = approx.residual_and_bound(f, ps, pl, k)
        assert np.abs((s[k] - c[k]) - R).max() <= 1e-10 * np.abs(c[k]).max()


def test_snr_grows_with_min_width():
    """Fig. CoeffQual: below 8 bins visibly different, above 16 largely equal."""
    f = np.random.default_rng(7).standard_normal(2048)
    snr = {mw: approx.snr_db(f, *_pair("blackman_harris", mw)) for mw in (4, 8, 16, 32)}
    hi = min(snr[16], snr[32])  # "largely equivalent" from 16 on (not necessarily monotone)
    assert snr[4] < snr[8] < hi
    assert hi - snr[4] > 20.0


@pytest.mark.parametrize("window,mw,sf,raster", [("blackman_harris", 8, 0, 0), ("hann", 12.5, 0, 1),
                                                 ("blackman_harris", 8, 256, 0),
                                                 ("hann", 4, 512, 2)])
def test_host_plan_options_parity(window, mw, sf, raster):
    from paper_1210_0084_b200 import api
    L = 2048 if sf else 256
    args = (FS, 200.0, FS / 2, 6, L, 32, raster)
    p = api.Plan(*args, host_only=True, window=window, min_width=mw, sampled_from=sf)
    ref = cqplan.make_plan(*args, window=window, min_width=mw, sampled_from=sf or None)
    e = p.export()
    assert np.array_equal(e["lo"], [c.lo for c in ref.stored])
    assert np.array_equal(e["len"], [c.L for c in ref.stored])
    assert np.array_equal(e["M"], [c.M for c in ref.stored])
    np.testing.assert_allclose(e["g"], np.concatenate([c.g for c in ref.stored]), rtol=0, atol=1e-12)


def test_host_plan_options_rejected():
    from paper_1210_0084_b200 import api
    args = (FS, 200.0, FS / 2, 6, 2048, 32, 0)
    for kw in (dict(min_width=0.5), dict(sampled_from=300), dict(sampled_from=4096),
               dict(window="kaiser")):
        with pytest.raises(Exception):
            api.Plan(*args, host_only=True, **kw)


def test_prop4_identity_complex_signal_all_channels():
    """Set 1 is complex: the identity over all 2K+2 channels, mirrors included."""
    from oracle.nsgt import analysis
    from oracle.slicq import forward_complex, offsets_full
    ps, pl = _pair("blackman_harris", 8)
    r = np.random.default_rng(13)
    f = r.standard_normal(pl.sl_len) + 1j * r.standard_normal(pl.sl_len)
    L, N2 = pl.sl_len, ps.sl_len
    c = [ck * approx.p4_scale(ch.M, L) for ck, ch in zip(analysis(f, pl.full, L), pl.full)]
    s = approx._two_layer_sum(forward_complex(f[None], ps)[0], ps.full, offsets_full(ps), L, N2)
    K = ps.layout.K
    for k in (0, 2, K + 1, K + 2, 2 * K + 1):
        sk = s[k] * approx.p4_scale(ps.full[k].M, N2)
        R, bound = approx.residual_and_bound(f, ps, pl, k, full=True)
        assert np.abs((sk - c[k]) - R).max() <= 1e-10 * np.abs(c[k]).max(), k
        assert np.all(np.abs(R) <= bound * (1 + 1e-12)), k
    sums = approx.channel_sums_complex(f, ps, pl)
    assert sums.shape == (2 * K + 2, 2)
