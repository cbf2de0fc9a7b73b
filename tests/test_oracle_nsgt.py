"""Pins for oracle/nsgt.py (Alg. 1/2) and oracle/direct.py against the paper's definitions."""
import numpy as np
import pytest

from oracle import cqplan, direct, nsgt
from oracle.cqplan import Channel

# Small CQ systems at lengths where brute force is cheap.  (fs, fmin, fmax, B, Ls, tr)
SMALL = [
    (8000.0, 200.0, 2000.0, 12, 128, 16),
    (8000.0, 300.0, None, 6, 96, 8),      # Ls not a power of two: rational a_k
    (44100.0, 500.0, None, 3, 160, 20),
    (22050.0, 100.0, 8000.0, 4, 256, 32),
]


def _plan(cfg):
    fs, fmin, fmax, B, Ls, tr = cfg
    return cqplan.make_plan(fs, fmin, fmax, B, Ls, tr, 0)


def test_numpy_fft_conventions_against_explicit_sums():
    # C1: FFT unnormalized with e^{-2 pi i}, IFFT with e^{+2 pi i} and 1/n (MATLAB/NumPy)
    rng = np.random.default_rng(1)
    for n in (4, 6, 10, 12, 30, 48):
        x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        k = np.arange(n)
        F = np.exp(-2j * np.pi * np.outer(k, k) / n)
        np.testing.assert_allclose(np.fft.fft(x), F @ x, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(np.fft.ifft(x), np.conj(F) @ x / n, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("cfg", SMALL)
def test_analysis_equals_direct_inner_products(cfg):
    # eq:CQ_coeff: c_{n,k} = <f, phi_{n,k}> for every (n, k), complex input,
    # all 2K+2 channels; <= 1e-10 (north_star)
    p = _plan(cfg)
    Ls = p.sl_len
    rng = np.random.default_rng(7)
    f = rng.standard_normal(Ls) + 1j * rng.standard_normal(Ls)
    c_fft = nsgt.analysis(f, p.full, Ls)
    c_dir = direct.coefficients(f, p.full, Ls)
    scale = max(np.max(np.abs(c)) for c in c_dir)
    for a, b in zip(c_fft, c_dir):
        assert np.max(np.abs(a - b)) <= 1e-10 * scale


@pytest.mark.parametrize("cfg", SMALL)
def test_frame_operator_is_diagonal(cfg):
    # Prop. 2 proof: brute-force S = sum phi phi^H equals the Fourier
    # multiplier by D = sum_k |g_k|^2 (C16 weights): S = F^H diag(D) F
    p = _plan(cfg)
    Ls = p.sl_len
    S_bf = direct.frame_operator(p.full, Ls)
    F = np.exp(-2j * np.pi * np.outer(np.arange(Ls), np.arange(Ls)) / Ls)
    S_diag = np.conj(F).T @ np.diag(p.D) @ F
    assert np.max(np.abs(S_bf - S_diag)) <= 1e-10 * Ls


@pytest.mark.parametrize("cfg", SMALL[:2])
def test_synthesis_is_canonical_dual_frame(cfg):
    # eq:candual: the Alg. 2 synthesis operator with g~ equals
    # S^{-1} Phi^* computed by brute force (Phi~ Phi^* = I)
    p = _plan(cfg)
    Ls = p.sl_len
    A = direct.analysis_matrix(p.full, Ls)          # rows phi^H
    S = A.conj().T @ A
    dual_atoms = np.linalg.solve(S, A.conj().T)     # columns S^-1 phi
    # apply Alg. 2 to unit coefficient vectors
    sizes = [c.M for c in p.full]
    offs = np.concatenate([[0], np.cumsum(sizes)])
    cols = []
    for i in range(offs[-1]):
        coeffs = [np.zeros(M, complex) for M in sizes]
        k = np.searchsorted(offs, i, side="right") - 1
        coeffs[k][i - offs[k]] = 1.0
        cols.append(nsgt.synthesis(coeffs, p.full, p.dual_full, Ls))
    Syn = np.array(cols).T
    assert np.max(np.abs(Syn - dual_atoms)) <= 1e-12 * max(1.0, np.max(np.abs(dual_atoms)))
    # and dual synthesis after analysis is the identity
    assert np.max(np.abs(Syn @ A - np.eye(Ls))) <= 1e-12


@pytest.mark.parametrize("Ls", [96, 128, 384, 1024, 3 * 1024, 1 << 14])
def test_full_length_perfect_reconstruction(Ls):
    # Prop. 1: iCQ-NSGT(CQ-NSGT(f)) = f, <= 1e-10, complex signals
    p = cqplan.make_plan(44100.0, 100.0, None, 12, Ls, 8, 0)
    rng = np.random.default_rng(Ls)
    for _ in range(3):
        f = rng.standard_normal(Ls) + 1j * rng.standard_normal(Ls)
        c = nsgt.analysis(f, p.full, Ls)
        fr = nsgt.synthesis(c, p.full, p.dual_full, Ls)
        assert np.linalg.norm(fr - f) / np.linalg.norm(f) <= 1e-10


def test_tight_frame_special_case():
    # north_star / P:135 footnote: a bank with sum_k |g_k|^2 == C constant is tight:
    # dual = g / C and sum_k ||c_k||^2 = C * Ls * ||f||^2 (unnormalized Parseval).
    Ls, h, C = 64, 8, 2.5
    chans = []
    for k in range(Ls // h):
        j = np.arange(k * h - h, k * h + h + 1)
        g = np.sqrt(C) * np.cos(np.pi * (j - k * h) / (2 * h))  # sin/cos pair at 50 % overlap
        chans.append(Channel(int(j[0]), g, 2 * h + 2))
    D = cqplan.frame_diagonal(chans, Ls)
    np.testing.assert_allclose(D, C, rtol=1e-14)
    duals = cqplan.canonical_dual(chans, D)
    for ch, gd in zip(chans, duals):
        np.testing.assert_allclose(gd, ch.g / C, rtol=1e-14)
    rng = np.random.default_rng(3)
    f = rng.standard_normal(Ls) + 1j * rng.standard_normal(Ls)
    c = nsgt.analysis(f, chans, Ls)
    energy = sum(np.vdot(ck, ck).real for ck in c)
    assert abs(energy - C * Ls * np.vdot(f, f).real) <= 1e-10 * energy
    fr = nsgt.synthesis(c, chans, duals, Ls)
    assert np.linalg.norm(fr - f) <= 1e-12 * np.linalg.norm(f)


@pytest.mark.parametrize("cfg", SMALL)
def test_per_channel_energy_identity(cfg):
    # follows from P:608-622: sum_n |c_{n,k}|^2 = sum_{j in J_k} |X[j]|^2 g_k[j]^2
    p = _plan(cfg)
    Ls = p.sl_len
    rng = np.random.default_rng(11)
    f = rng.standard_normal(Ls)
    X = np.fft.fft(f)
    c = nsgt.analysis(f, p.full, Ls)
    for ch, ck in zip(p.full, c):
        e = np.sum(np.abs(X[np.mod(ch.bins, Ls)]) ** 2 * ch.g ** 2)
        assert abs(np.vdot(ck, ck).real - e) <= 1e-12 * max(e, 1.0)


@pytest.mark.parametrize("cfg", SMALL)
def test_real_input_symmetries(cfg):
    # Table 1 symmetry for real f (reading C15): mirror relation,
    # DC coefficients real, Nyquist coefficients times e^{-i pi Ls n / M} real
    p = _plan(cfg)
    Ls = p.sl_len
    K = p.layout.K
    rng = np.random.default_rng(5)
    f = rng.standard_normal(Ls)
    c = nsgt.analysis(f, p.full, Ls)
    mir = nsgt.mirror_coeffs(c[:K + 2], p)
    scale = max(np.max(np.abs(x)) for x in c)
    for a, b in zip(c[K + 2:], mir):
        assert np.max(np.abs(a - b)) <= 1e-12 * scale
    assert np.max(np.abs(c[0].imag)) <= 1e-12 * scale
    M = p.stored[K + 1].M
    ny = c[K + 1] * np.exp(-1j * np.pi * Ls * np.arange(M) / M)
    assert np.max(np.abs(ny.imag)) <= 1e-12 * scale
    # real-mode synthesis reconstructs (imaginary part vanishes)
    re, im = nsgt.synthesis_real(c[:K + 2], p, return_imag=True)
    assert np.linalg.norm(re - f) <= 1e-12 * np.linalg.norm(f)
    assert np.linalg.norm(im) <= 1e-12 * np.linalg.norm(f)


def test_real_mode_synthesis_is_hermitian_projection():
    # For MODIFIED coefficients, real-mode synthesis = Re(full synthesis) when the mirrors
    # are regenerated from C15 — and it is linear in the stored coefficients.
    p = _plan(SMALL[0])
    Ls = p.sl_len
    K = p.layout.K
    rng = np.random.default_rng(9)
    cs = [rng.standard_normal(ch.M) + 1j * rng.standard_normal(ch.M) for ch in p.stored]
    full = cs + nsgt.mirror_coeffs(cs, p)
    ref = nsgt.synthesis(full, p.full, p.dual_full, Ls).real
    np.testing.assert_allclose(nsgt.synthesis_real(cs, p), ref, rtol=0, atol=1e-14)
    cs2 = [rng.standard_normal(ch.M) + 1j * rng.standard_normal(ch.M) for ch in p.stored]
    lin = nsgt.synthesis_real([a + 2 * b for a, b in zip(cs, cs2)], p)
    np.testing.assert_allclose(lin, nsgt.synthesis_real(cs, p) + 2 * nsgt.synthesis_real(cs2, p),
                               atol=1e-12)
