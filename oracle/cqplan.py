"""ORACLE (test infrastructure only) — the plan of the CQ-NSGT / sliCQ in float64.

Everything here is the paper's construction written out directly:
  * Table 1 layout and the constant Q ............ P:242-260 (readings C3, C4)
  * sampled Hann filters g_k and plateaus ........ P:262 (readings C7, C8)
  * Blackman-Harris filters, minimal width,
    filters sampled from a length-L system ....... P:377-386 (Prop. 4), P:475-490 (C20-C22)
  * coefficient counts M_k = L/a_k >= L_k ........ P:168-170, P:264-265 (C9, C10)
  * frame diagonal and canonical dual ............ P:219-228, Prop. 2 (C1, C16)
  * Tukey slicing window h_0 and its dual ........ P:353-356, P:363-374 (C11, C12)

A *channel* is ``Channel(lo, g, M)``: the filter g_k sampled on the contiguous,
UNWRAPPED integer bin interval J_k = [lo, lo+len(g)) of a length-Ls DFT
(reading C5: supports are never reduced mod Ls before folding), plus its
coefficient count M = Ls/a_k.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

EDGE_EPS = 1e-9   # C7/C18: support-edge guard
K_EPS = 1e-12     # C4/C18: guard on B*log2(.)
MIN_WIDTH = 4.0   # C7: minimum filter width in bins


@dataclass
class Channel:
    lo: int                 # first bin of J_k (may be negative: DC plateau, C5)
    g: np.ndarray           # float64 filter values on J_k
    M: int                  # coefficient count L/a_k
    kind: str = "cq"        # "dc", "cq", "nyq", "mirror"
    partner: int = -1       # for mirrors: the stored channel k it mirrors

    @property
    def L(self) -> int:
        return int(self.g.shape[0])

    @property
    def bins(self) -> np.ndarray:
        return np.arange(self.lo, self.lo + self.L)


@dataclass
class Layout:
    K: int
    Q: float
    xi: np.ndarray       # xi_1..xi_K  (Hz)
    Omega: np.ndarray    # Omega_1..Omega_K (Hz)
    fs: float


@dataclass
class Plan:
    fs: float
    fmin: float
    fmax: float
    B: int
    sl_len: int          # 2N
    tr: int              # transition length ("M" in P:373)
    rasterize: int
    layout: Layout
    stored: List[Channel]          # channels 0..K+1 (DC, CQ 1..K, Nyquist) — what real input stores
    full: List[Channel]            # all 2K+2 channels of Table 1 (stored + mirrors K+2..2K+1)
    D: np.ndarray                  # frame diagonal on [0, 2N)  (P:221-223 weights per C1/C16)
    dual_stored: List[np.ndarray]  # dual filter values on each stored channel's J_k
    dual_full: List[np.ndarray]
    h0: np.ndarray                 # h_0[t], t = -N..N-1  (index t+N)
    h0dual: np.ndarray             # canonical dual slicing window, same indexing
    painless: bool = True          # M_k >= L_k for every channel (False only for sampled_from)

    @property
    def N(self) -> int:
        return self.sl_len // 2

    @property
    def M(self) -> np.ndarray:
        return np.array([c.M for c in self.stored], dtype=np.int64)

    @property
    def coeffs_per_slice(self) -> int:
        return int(sum(c.M for c in self.stored))


# ---------------------------------------------------------------- Table 1 layout
def q_factor(B: int) -> float:
    """Q = xi_k / Omega_k = (2^(1/B) - 2^(-1/B))^-1."""
    return 1.0 / (2.0 ** (1.0 / B) - 2.0 ** (-1.0 / B))


def cq_layout(fs: float, fmin: float, fmax: Optional[float], B: int) -> Layout:
    """Centre frequencies xi_k = xi_min 2^((k-1)/B), k = 1..K and Omega_k = xi_k/Q
    (Table 1; Omega for k = 1, K and 2..K-1 coincide, reading C3).

    K (reading C4): the paper asks xi_max <= xi_K < fs/2, impossible when
    fmax >= fs/2, so K = min(smallest k with xi_k >= xi_max, largest k with xi_k < fs/2).
    """
    if fmax is None:
        fmax = fs / 2.0
    if not (fs > 0 and 0 < fmin < fs / 2 and fmax > fmin and B >= 1):
        raise ValueError("invalid CQ parameters")
    y = B * math.log2(fmax / fmin)
    k_cover = math.ceil(y - K_EPS) + 1          # smallest k: (k-1) >= y
    x = B * math.log2((fs / 2.0) / fmin)
    k_nyq = math.ceil(x - K_EPS)                # largest k: (k-1) < x
    K = min(k_cover, k_nyq)
    if K < 1:
        raise ValueError("K < 1")
    Q = q_factor(B)
    k = np.arange(1, K + 1, dtype=np.float64)
    xi = fmin * 2.0 ** ((k - 1) / B)
    return Layout(K=K, Q=Q, xi=xi, Omega=xi / Q, fs=fs)


# ---------------------------------------------------------------- filters
def hann(x: np.ndarray) -> np.ndarray:
    """H(x) = cos^2(pi x) on |x| <= 1/2, 0 outside (reading C7 of P:262's H)."""
    x = np.asarray(x, dtype=np.float64)
    return np.where(np.abs(x) <= 0.5, np.cos(np.pi * np.clip(x, -0.5, 0.5)) ** 2, 0.0)


# 4-term Blackman-Harris (the window of the paper's approximation experiments),
# centred on [-1/2, 1/2] (reading C20): H(x) = a0 + a1 cos 2 pi x + a2 cos 4 pi x + a3 cos 6 pi x
BH = (0.35875, 0.48829, 0.14128, 0.01168)


def blackman_harris(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    a0, a1, a2, a3 = BH
    v = a0 + a1 * np.cos(2 * np.pi * x) + a2 * np.cos(4 * np.pi * x) + a3 * np.cos(6 * np.pi * x)
    return np.where(np.abs(x) <= 0.5, v, 0.0)


WINDOWS = {"hann": hann, "blackman_harris": blackman_harris}


def cq_filter(xi: float, Om: float, fs: float, Ls: int, window: str = "hann",
              min_width: float = MIN_WIDTH, grid: Optional[int] = None):
    """g_k[j] = H((j fs/Ls - xi_k)/Omega_k) with width clamp (reading C7).

    omega = xi Ls/fs (fractional), W = max(Omega Ls/fs, min_width) bins,
    J = [ceil(omega - W/2 - eps), floor(omega + W/2 + eps)], g = H((j - omega)/W).
    grid = 2N (Prop. 4, reading C21): the filter of a length-Ls system whose samples at the
    multiples of s = Ls/2N are the length-2N system's filter, g_k[j] = g^L_k[j Ls/2N]:
    omega = s (xi 2N/fs), W = s max(Omega 2N/fs, min_width) -- the width clamp acts on the
    2N grid.  Returns (lo, g, omega, W)."""
    if grid is None:
        omega = xi * Ls / fs
        W = max(Om * Ls / fs, min_width)
    else:
        sc = Ls // grid
        omega = sc * (xi * grid / fs)
        W = sc * max(Om * grid / fs, min_width)
    lo = math.ceil(omega - W / 2 - EDGE_EPS)
    hi = math.floor(omega + W / 2 + EDGE_EPS)
    j = np.arange(lo, hi + 1, dtype=np.float64)
    return lo, WINDOWS[window]((j - omega) / W), omega, W


def _eval_on(lo: int, g: np.ndarray, j: np.ndarray) -> np.ndarray:
    """Filter value at integer bins j (0 off the support J)."""
    idx = j - lo
    ok = (idx >= 0) & (idx < g.shape[0])
    out = np.zeros(j.shape, dtype=np.float64)
    out[ok] = g[idx[ok]]
    return out


def plateau_filters(cq, Ls: int):
    """Plateaus g_0 (DC) and g_{K+1} (Nyquist) (Table 1 rows 0 and K+1; reading C8).

    g_0(j) = 1 - g_1(|j|) on J_0 = [-floor(omega_1), floor(omega_1)]
    g_{K+1}(j) = max(0, 1 - g_K(j) - g_K(Ls - j)) on [ceil(omega_K), floor(Ls - omega_K)]."""
    lo1, g1, om1, _ = cq[0]
    loK, gK, omK, _ = cq[-1]
    a = math.floor(om1)
    j0 = np.arange(-a, a + 1)
    g0 = 1.0 - _eval_on(lo1, g1, np.abs(j0))
    b0, b1 = math.ceil(omK), math.floor(Ls - omK)
    jn = np.arange(b0, b1 + 1)
    gn = np.maximum(0.0, 1.0 - _eval_on(loK, gK, jn) - _eval_on(loK, gK, Ls - jn))
    return (-a, g0), (b0, gn)


# ---------------------------------------------------------------- coefficient counts
def is_235_smooth(m: int) -> bool:
    for p in (2, 3, 5):
        while m % p == 0:
            m //= p
    return m == 1


def smallest_even_smooth_ge(L: int) -> int:
    """Smallest even 2/3/5-smooth integer >= L (reading C9 of P:264-265)."""
    m = max(2, L)
    while True:
        if m % 2 == 0 and is_235_smooth(m):
            return m
        m += 1


def channel_lengths(Ls_list: List[int], B: int, rasterize: int) -> List[int]:
    """M_k for the stored channels 0..K+1 (reading C9/C10; P:546-548 for rasterization).

    rasterize 0: each M_k = smallest even smooth >= L_k.
    rasterize 2 (full): one M >= max_k L_k for every channel ("L/a_k constant").
    rasterize 1 (per octave): groups {0}, {K+1}, CQ octaves floor((k-1)/B)."""
    K = len(Ls_list) - 2
    if rasterize == 0:
        return [smallest_even_smooth_ge(L) for L in Ls_list]
    if rasterize == 2:
        m = smallest_even_smooth_ge(max(Ls_list))
        return [m] * (K + 2)
    if rasterize == 1:
        out = [0] * (K + 2)
        out[0] = smallest_even_smooth_ge(Ls_list[0])
        out[K + 1] = smallest_even_smooth_ge(Ls_list[K + 1])
        groups = {}
        for k in range(1, K + 1):
            groups.setdefault((k - 1) // B, []).append(k)
        for ks in groups.values():
            m = smallest_even_smooth_ge(max(Ls_list[k] for k in ks))
            for k in ks:
                out[k] = m
        return out
    raise ValueError("rasterize must be 0, 1 or 2")


# ---------------------------------------------------------------- painless dual
def frame_diagonal(channels: List[Channel], Ls: int) -> np.ndarray:
    """D[j] = sum over ALL channels of |g_k[j]|^2, j in [0, Ls)  (Prop. 2 / P:221-223,
    unweighted per readings C1/C16).  Unwrapped supports are accumulated mod Ls."""
    D = np.zeros(Ls, dtype=np.float64)
    for c in channels:
        np.add.at(D, np.mod(c.bins, Ls), c.g ** 2)
    return D


def canonical_dual(channels: List[Channel], D: np.ndarray) -> List[np.ndarray]:
    """g~_k = g_k / D  (eq:painlessframe2 with the C1 weighting)."""
    Ls = D.shape[0]
    if np.any(D <= 0):
        raise ValueError("not a frame: frame diagonal has zeros (P:221)")
    return [c.g / D[np.mod(c.bins, Ls)] for c in channels]


# ---------------------------------------------------------------- slicing windows
def tukey_slicing_window(N: int, tr: int) -> np.ndarray:
    """h_0[t], t = -N..N-1 (returned at index t+N): Tukey window of essential length N,
    transitions of length tr, zero-padded to 2N (reading C11):
      1                                   |t| <= (N-tr)/2
      cos^2(pi (|t| - (N-tr)/2) / (2 tr))  (N-tr)/2 < |t| < (N+tr)/2
      0                                   otherwise."""
    t = np.abs(np.arange(-N, N, dtype=np.float64))
    a, b = (N - tr) / 2.0, (N + tr) / 2.0
    h = np.zeros(2 * N, dtype=np.float64)
    h[t <= a] = 1.0
    m = (t > a) & (t < b)
    h[m] = np.cos(np.pi * (t[m] - a) / (2.0 * tr)) ** 2
    return h


def periodize(h: np.ndarray, N: int) -> np.ndarray:
    """sum_m T_{mN} h on one period of length N (h indexed t+N, t in [-N, N))."""
    out = np.zeros(N, dtype=np.float64)
    t = np.arange(-N, N)
    np.add.at(out, np.mod(t, N), h)
    return out


def dual_slicing_window(h0: np.ndarray, N: int) -> np.ndarray:
    """Canonical dual h~_0 = h_0 / sum_m T_{mN} h_0^2, so that sum_m T_{mN}(h_0 h~_0) == 1
    (dualwincond; reading C12)."""
    den = periodize(h0 * h0, N)
    t = np.arange(-N, N)
    return h0 / den[np.mod(t, N)]


# ---------------------------------------------------------------- the plan
def _raw_filters(lay: Layout, fs: float, Ls: int, window: str, min_width: float,
                 grid: Optional[int]):
    cq = [cq_filter(lay.xi[i], lay.Omega[i], fs, Ls, window, min_width, grid)
          for i in range(lay.K)]
    (lo0, g0), (loN, gN) = plateau_filters(cq, Ls)
    return [(lo0, g0, "dc")] + [(lo, g, "cq") for (lo, g, _, _) in cq] + [(loN, gN, "nyq")]


def make_plan(fs: float, fmin: float, fmax: Optional[float], B: int, sl_len: int, tr: int,
              rasterize: int = 0, window: str = "hann", min_width: float = MIN_WIDTH,
              sampled_from: Optional[int] = None) -> Plan:
    """Precompute everything Alg. 3/4 need for slices of length 2N = sl_len.

    window: "hann" or "blackman_harris"; min_width: the lower bound on
    the filter width in bins (C7; the x axis of the paper's Fig. CoeffQual).
    sampled_from = 2N' (Prop. 4; reading C21): the length-sl_len system whose
    filters, sampled every sl_len/2N' bins, are those of the length-2N' system with the same
    parameters, and whose counts are M_k = (sl_len/2N') M'_k (the same hops a_k) -- the
    full-length CQ-NSGT that the sliCQ with slices 2N' approximates."""
    if sl_len % 4 != 0 or not is_235_smooth(sl_len):
        raise ValueError("sl_len must be divisible by 4 and 2/3/5-smooth")
    N = sl_len // 2
    if tr % 2 != 0 or tr < 2 or tr >= N:
        raise ValueError("tr_area must be even, >= 2 and < sl_len/2 (P:373: M < N)")
    if not min_width >= 1.0:
        raise ValueError("min_width must be >= 1 bin")
    lay = cq_layout(fs, fmin, fmax, B)
    Ls = sl_len
    if sampled_from is not None and (sampled_from <= 0 or Ls % sampled_from != 0):
        raise ValueError("sampled_from must divide sl_len")
    raw = _raw_filters(lay, fs, Ls, window, min_width, sampled_from)
    if sampled_from is None:
        Ms = channel_lengths([g.shape[0] for _, g, _ in raw], B, rasterize)
    else:
        raw0 = _raw_filters(lay, fs, sampled_from, window, min_width, None)
        Ms = [(Ls // sampled_from) * m
              for m in channel_lengths([g.shape[0] for _, g, _ in raw0], B, rasterize)]
    stored = [Channel(lo, g, M, kind) for (lo, g, kind), M in zip(raw, Ms)]
    painless = all(c.M >= c.L for c in stored)
    # a sampled_from system keeps the slice system's hops even where its support is longer
    # than M_k (Prop. 4 needs only the analysis, which Alg. 1 folds; reading C21)
    if not painless and sampled_from is None:
        raise ValueError("painless condition M_k >= L_k violated (P:170)")
    K = lay.K
    # mirrors K+2..2K+1 of Table 1: channel 2K+2-k mirrors k = K..1 about Nyquist
    mirrors = []
    for kk in range(K + 2, 2 * K + 2):
        k = 2 * K + 2 - kk
        c = stored[k]
        mirrors.append(Channel(Ls - (c.lo + c.L - 1), c.g[::-1].copy(), c.M, "mirror", k))
    full = stored + mirrors
    D = frame_diagonal(full, Ls)
    dual_full = canonical_dual(full, D)
    h0 = tukey_slicing_window(N, tr)
    return Plan(fs=fs, fmin=fmin, fmax=fs / 2 if fmax is None else fmax, B=B, sl_len=sl_len,
                tr=tr, rasterize=rasterize, layout=lay, stored=stored, full=full, D=D,
                dual_stored=dual_full[:K + 2], dual_full=dual_full, h0=h0,
                h0dual=dual_slicing_window(h0, N), painless=painless)
