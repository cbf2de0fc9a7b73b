"""ORACLE (test infrastructure only) — painless NSG analysis/synthesis, Alg. 1 and Alg. 2.

FFT conventions (reading C1): the paper's platform (MATLAB/NumPy) —
FFT_n unnormalized, IFFT_n including 1/n.  With these, Alg. 1 line P:188 is
``c_k = sqrt(M_k) * ifft(fold(fft(f) * g_k))`` and Alg. 2 line P:200 is
``f_k = fft(c_k) / sqrt(M_k)``; the matching dual is g_k / sum_l |g_l|^2.

``numpy.fft`` (pocketfft) is the FFT primitive; it is pinned against explicit
DFT sums in tests/test_oracle_nsgt.py.
"""
from __future__ import annotations

from typing import List, Sequence

import numpy as np

from .cqplan import Channel, Plan


def analysis(f: np.ndarray, channels: Sequence[Channel], Ls: int) -> List[np.ndarray]:
    """Alg. 1: c = CQ-NSGT_Ls(f, g, a).

    X = FFT_Ls(f)
    buf[j mod M_k] += X[j mod Ls] * conj(g_k[j])    for j in J_k (unwrapped, C5)
    c_k = sqrt(M_k) * IFFT_{M_k}(buf)
    """
    f = np.asarray(f)
    assert f.shape == (Ls,)
    X = np.fft.fft(f.astype(np.complex128))
    out = []
    for c in channels:
        buf = np.zeros(c.M, dtype=np.complex128)
        j = c.bins
        np.add.at(buf, np.mod(j, c.M), X[np.mod(j, Ls)] * np.conj(c.g))
        out.append(np.sqrt(c.M) * np.fft.ifft(buf))
    return out


def synthesis(coeffs: Sequence[np.ndarray], channels: Sequence[Channel],
              duals: Sequence[np.ndarray], Ls: int) -> np.ndarray:
    """Alg. 2: f~ = iCQ-NSGT_Ls(c, g~, a).

    f_k = sqrt(a_k/Ls) FFT_{M_k}(c_k) = FFT(c_k)/sqrt(M_k)
    F[j mod Ls] += f_k[j mod M_k] * g~_k[j]
    f~ = IFFT_Ls(F)
    """
    F = np.zeros(Ls, dtype=np.complex128)
    for c, ck, gd in zip(channels, coeffs, duals):
        fk = np.fft.fft(np.asarray(ck, dtype=np.complex128)) / np.sqrt(c.M)
        j = c.bins
        np.add.at(F, np.mod(j, Ls), fk[np.mod(j, c.M)] * gd)
    return np.fft.ifft(F)


# ------------------------------------------------------------------ real-input mode
def mirror_coeffs(stored: Sequence[np.ndarray], plan: Plan) -> List[np.ndarray]:
    """Coefficients of the mirror channels K+2..2K+1 of a REAL input, regenerated from
    the stored channels 1..K (reading C15; Table 1 symmetry P:252):
        c_{n, 2K+2-k} = exp(2 pi i Ls n / M_k) * conj(c_{n,k})."""
    K = plan.layout.K
    Ls = plan.sl_len
    out = []
    for kk in range(K + 2, 2 * K + 2):
        k = 2 * K + 2 - kk
        M = plan.stored[k].M
        n = np.arange(M)
        out.append(np.exp(2j * np.pi * Ls * n / M) * np.conj(np.asarray(stored[k], np.complex128)))
    return out


def analysis_real(f: np.ndarray, plan: Plan) -> List[np.ndarray]:
    """Stored channels 0..K+1 of a real length-2N frame (the GPU's output set)."""
    return analysis(np.asarray(f, np.float64), plan.stored, plan.sl_len)


def synthesis_real(stored: Sequence[np.ndarray], plan: Plan, return_imag: bool = False):
    """Real-mode synthesis: regenerate the mirrors (C15), run the full 2K+2-channel
    Alg. 2, and keep the real part.  For coefficients of a real signal the imaginary
    part vanishes; for modified coefficients this is the Hermitian projection."""
    full = list(stored) + mirror_coeffs(stored, plan)
    f = synthesis(full, plan.full, plan.dual_full, plan.sl_len)
    if return_imag:
        return f.real, f.imag
    return f.real
