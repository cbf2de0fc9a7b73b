"""ORACLE (test infrastructure only) — sliCQ vs full-length CQ-NSGT, Prop. 4
and the approximation experiment of Sec. V-A.

  full-length system G(g^L, a): cqplan.make_plan(..., sl_len=L, sampled_from=2N) -- its
      filters sampled every L/2N bins are the slice system's, g_k[j] = g^L_k[jL/2N]
      (P:381-383), and its hops a_k are the slice system's (M^L_k = (L/2N) M_k)
  c = CQ-NSGT_L(f) (Alg. 1); s = sliCQ two-layer array (Alg. 3)
  s^0 + s^1 - c = R[n] (proof), bounded by eq:inner_outer
  SNR = 20 log10(||c|| / ||c - (s^0 + s^1)||)

Normalisation (reading C22): Prop. 4 and its proof use c_{n,k} = <f, T_{n a_k} g^L_k-check>
with g-check = F^{-1} g the NON-unitary inverse DFT (1/L sum_j g[j] e^{2 pi i j l / L}) --
the only normalisation under which g_k-check is the plain periodisation of g^L_k-check
(P:644-647).  The library / Alg. 1 coefficients (reading C1) are sqrt(L a_k) times these
(sqrt(2N a_k) for a slice), so everything here is compared after p4_scale.

Real input: the library's path is real-input (C15), so the experiment runs on real signals
over the stored channels 0..K+1 (the paper's Set 1 is complex; reading C23).
"""
from __future__ import annotations

from typing import List

import numpy as np

from .cqplan import Plan
from .nsgt import analysis_real
from .slicq import forward as slicq_forward, two_layer


def p4_scale(M: int, length: int) -> float:
    """Alg. 1 coefficient -> Prop. 4 coefficient: c_P4 = c sqrt(M)/length (= c / sqrt(length a_k))."""
    return float(np.sqrt(M)) / float(length)


def check_pair(plan_s: Plan, plan_L: Plan) -> int:
    """The systems of Prop. 4: same channels, L a multiple of 2N, M^L_k = (L/2N) M_k."""
    L, N2 = plan_L.sl_len, plan_s.sl_len
    if L % N2:
        raise ValueError("L must be a multiple of the slice length")
    sc = L // N2
    if len(plan_L.stored) != len(plan_s.stored):
        raise ValueError("channel counts differ")
    for a, b in zip(plan_s.stored, plan_L.stored):
        if b.M != sc * a.M:
            raise ValueError("full-length counts are not (L/2N) M_k")
    return sc


def slice_sum(f: np.ndarray, plan_s: Plan, L: int) -> List[np.ndarray]:
    """(s^0 + s^1)_k for every stored channel, from Alg. 3's two-layer array, P4-normalised."""
    c = slicq_forward(f[None], plan_s)[0]             # [S][C]
    s = two_layer(c, plan_s, L)
    return [(sk[0] + sk[1]) * p4_scale(ch.M, plan_s.sl_len) for sk, ch in zip(s, plan_s.stored)]


def full_coeffs(f: np.ndarray, plan_L: Plan) -> List[np.ndarray]:
    """c_k of the full-length CQ-NSGT (Alg. 1 at length L), P4-normalised."""
    return [ck * p4_scale(ch.M, plan_L.sl_len) for ck, ch in zip(analysis_real(f, plan_L), plan_L.stored)]


def snr_db(f: np.ndarray, plan_s: Plan, plan_L: Plan) -> float:
    """20 log10(||c|| / ||c - (s^0 + s^1)||) over the stored channels."""
    check_pair(plan_s, plan_L)
    L = plan_L.sl_len
    c = full_coeffs(f, plan_L)
    s = slice_sum(f, plan_s, L)
    num = sum(float(np.sum(np.abs(ck) ** 2)) for ck in c)
    den = sum(float(np.sum(np.abs(ck - sk) ** 2)) for ck, sk in zip(c, s))
    return 10.0 * np.log10(num / den)


def channel_sums(f: np.ndarray, plan_s: Plan, plan_L: Plan) -> np.ndarray:
    """Per stored channel: [sum |c|^2, sum |c - (s^0 + s^1)|^2] (P4 normalisation)."""
    c = full_coeffs(f, plan_L)
    s = slice_sum(f, plan_s, plan_L.sl_len)
    return np.array([[np.sum(np.abs(ck) ** 2), np.sum(np.abs(ck - sk) ** 2)] for ck, sk in zip(c, s)])


# ------------------------------------------------------------------ complex input (Set 1)
def _two_layer_sum(c_rows: np.ndarray, chans, off, L: int, N2: int) -> List[np.ndarray]:
    """s^0 + s^1 per channel from slice rows c[S][...] (Alg. 3 lines P:320-323, any layout)."""
    S = c_rows.shape[0]
    out = []
    for k, ch in enumerate(chans):
        M = ch.M
        width = L * M // N2
        s = np.zeros((2, width), dtype=np.complex128)
        for m in range(S):
            idx = np.mod((m - 1) * (M // 2) + np.arange(M), width)
            s[m % 2, idx] = c_rows[m, off[k]:off[k + 1]]
        out.append(s[0] + s[1])
    return out


def channel_sums_complex(f: np.ndarray, plan_s: Plan, plan_L: Plan) -> np.ndarray:
    """Complex f (the paper's Set 1): per channel of all 2K+2 (Table-1 order)
    [sum |c|^2, sum |c - (s^0 + s^1)|^2], P4-normalised (C22)."""
    from .nsgt import analysis
    from .slicq import forward_complex, offsets_full
    check_pair(plan_s, plan_L)
    L, N2 = plan_L.sl_len, plan_s.sl_len
    f = np.asarray(f, np.complex128)
    c = [ck * p4_scale(ch.M, L) for ck, ch in zip(analysis(f, plan_L.full, L), plan_L.full)]
    rows = forward_complex(f[None], plan_s)[0]
    s = _two_layer_sum(rows, plan_s.full, offsets_full(plan_s), L, N2)
    s = [sk * p4_scale(ch.M, N2) for sk, ch in zip(s, plan_s.full)]
    return np.array([[np.sum(np.abs(ck) ** 2), np.sum(np.abs(ck - sk) ** 2)] for ck, sk in zip(c, s)])


# ------------------------------------------------------------------ Prop. 4, term by term
def atom(ch, L: int, x: float = 0.0) -> np.ndarray:
    """T_x g^L_k-check, g-check = F^{-1} g^L_k with the non-unitary inverse DFT (reading
    C22).  x may be fractional (a_k = L/M_k need not be an integer): the translate of the
    band-limited atom, F^{-1}(M_{-x} g)."""
    g = np.zeros(L, dtype=np.complex128)
    j = np.mod(ch.bins, L)
    np.add.at(g, j, ch.g * np.exp(-2j * np.pi * ch.bins * x / L))
    return np.fft.ifft(g)


def slicing_windows(plan_s: Plan, L: int, m: int) -> np.ndarray:
    """h_m = T_{mN} h_0 on Z_L (h_0 centred at 0)."""
    N = plan_s.sl_len // 2
    h = np.zeros(L)
    t = np.arange(-N, N)
    h[np.mod(t + m * N, L)] = plan_s.h0
    return h


def residual_and_bound(f: np.ndarray, plan_s: Plan, plan_L: Plan, k: int, full: bool = False):
    """For channel k and every n = m N/a_k + n^s: R[n] of the proof by direct
    inner products over C^L, and the right-hand side of eq:inner_outer.
    Returns (R, bound), both P4-normalised arrays of length L/a_k."""
    L = plan_L.sl_len
    N = plan_s.sl_len // 2
    sc = check_pair(plan_s, plan_L)
    ch = (plan_L.full if full else plan_L.stored)[k]  # full: all 2K+2 channels (complex f)
    M = ch.M
    a = L / M                                          # a_k (possibly fractional)
    half = (plan_s.full if full else plan_s.stored)[k].M // 2   # N / a_k
    nf = np.linalg.norm(f)
    R = np.zeros(M, dtype=np.complex128)
    bound = np.zeros(M)
    for n in range(M):
        m = n // half
        hs = slicing_windows(plan_s, L, m) + slicing_windows(plan_s, L, m + 1)
        main = atom(ch, L, n * a)                      # T_{n a_k} g-check, n a_k = n^s a_k + mN
        spill = np.zeros(L, dtype=np.complex128)
        for j in range(1, sc):
            spill += atom(ch, L, n * a + 2 * j * N)
        u = (1.0 - hs) * main
        v = hs * spill
        # s^0 + s^1 = <f, hs main> + <f, v> = c - <f, u> + <f, v>  (the proof prints "+" on
        # the first term of R[n]; the bound takes absolute values; reading C24)
        R[n] = -np.vdot(u, f) + np.vdot(v, f)         # <f, u> = sum_l f[l] conj(u[l])
        bound[n] = nf * (np.linalg.norm(u) + np.linalg.norm(v))
    return R, bound
