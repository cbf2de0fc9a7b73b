"""ORACLE (test infrastructure only) — the sliced CQ-NSGT, Alg. 3 / Alg. 4.

  padding to L, a multiple of 2N ............ P:299 (reading C13: zeros at the end)
  slice m: f^m[j] = f[((m-1)N + j) mod L] h_0[j-N]   P:316-318, circular indices P:328 (C14)
  c^m = CQ-NSGT_2N(f^m)  ..................... P:319 (typo f -> f^m, C2), Alg. 1
  two-layer array s^{m mod 2} ................ P:320-323
  synthesis + windowed overlap-add ........... P:336-346 (Alg. 4)

Coefficient layout returned here matches the library's: complex [batch][S][sum_k M_k],
channel k (k = 0..K+1) in columns [off_k, off_k + M_k).
"""
from __future__ import annotations

from typing import Iterable, List, Optional, Sequence

import numpy as np

from .cqplan import Plan
from .nsgt import analysis_real, synthesis_real


def padded_length(n: int, sl_len: int) -> int:
    """L = ceil(n / 2N) * 2N."""
    return -(-n // sl_len) * sl_len


def num_slices(n: int, sl_len: int) -> int:
    """S = L / N  (the loop bound of Alg. 3)."""
    return 2 * padded_length(n, sl_len) // sl_len


def offsets(plan: Plan) -> np.ndarray:
    return np.concatenate([[0], np.cumsum(plan.M)]).astype(np.int64)


def slice_frame(x: np.ndarray, m: int, plan: Plan, L: int) -> np.ndarray:
    """f^m[j] = f[((m-1)N + j) mod L] * h_0[j - N], j = 0..2N-1.
    ``x`` is the UNPADDED signal; positions >= len(x) are the zero padding."""
    N = plan.N
    idx = np.mod((m - 1) * N + np.arange(2 * N), L)
    v = np.zeros(2 * N, dtype=np.float64)
    ok = idx < x.shape[0]
    v[ok] = x[idx[ok]]
    return v * plan.h0


def concat(chans: Sequence[np.ndarray]) -> np.ndarray:
    return np.concatenate([np.asarray(c, np.complex128) for c in chans])


def split(row: np.ndarray, plan: Plan) -> List[np.ndarray]:
    off = offsets(plan)
    return [row[off[k]:off[k + 1]] for k in range(len(plan.stored))]


def forward(x: np.ndarray, plan: Plan, slices: Optional[Iterable[int]] = None) -> np.ndarray:
    """Alg. 3 for a batch of real signals x[batch][n] -> c[batch][S'][sum M_k]
    (S' = all S slices, or the requested subset in the given order)."""
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    B, n = x.shape
    L = padded_length(n, plan.sl_len)
    S = 2 * L // plan.sl_len
    ms = list(range(S)) if slices is None else list(slices)
    out = np.zeros((B, len(ms), plan.coeffs_per_slice), dtype=np.complex128)
    for b in range(B):
        for i, m in enumerate(ms):
            out[b, i] = concat(analysis_real(slice_frame(x[b], m, plan, L), plan))
    return out


def slice_contribution(c_row: np.ndarray, m: int, plan: Plan, L: int):
    """Alg. 4 body for one slice: positions ((m-1)N + j) mod L and values
    f~^m[j] h~_0[j-N]."""
    N = plan.N
    fm = synthesis_real(split(c_row, plan), plan)
    pos = np.mod((m - 1) * N + np.arange(2 * N), L)
    return pos, fm * plan.h0dual


def inverse(c: np.ndarray, plan: Plan, n: int) -> np.ndarray:
    """Alg. 4: c[batch][S][sum M_k] -> y[batch][n] (overlap-add, padding trimmed)."""
    c = np.asarray(c)
    if c.ndim == 2:
        c = c[None]
    B, S, _ = c.shape
    L = padded_length(n, plan.sl_len)
    assert S == 2 * L // plan.sl_len
    y = np.zeros((B, L), dtype=np.float64)
    for b in range(B):
        for m in range(S):
            pos, val = slice_contribution(c[b, m], m, plan, L)
            np.add.at(y[b], pos, val)
    return y[:, :n]


def inverse_samples(c_of: dict, plan: Plan, n: int, a: int, b: int) -> np.ndarray:
    """y[a:b] of one signal from only the slices that touch [a, b).
    ``c_of`` maps slice index m -> coefficient row (used for sampled parity at full size)."""
    N = plan.N
    L = padded_length(n, plan.sl_len)
    S = 2 * L // plan.sl_len
    y = np.zeros(b - a, dtype=np.float64)
    for m in needed_slices(a, b, plan, n):
        pos, val = slice_contribution(c_of[m], m, plan, L)
        sel = (pos >= a) & (pos < b)
        np.add.at(y, pos[sel] - a, val[sel])
    return y


def needed_slices(a: int, b: int, plan: Plan, n: int) -> List[int]:
    """Slices whose dual window h~_0 is nonzero somewhere on samples [a, b)."""
    N, tr = plan.N, plan.tr
    L = padded_length(n, plan.sl_len)
    S = 2 * L // plan.sl_len
    half = (N + tr) // 2  # h~_0[t] != 0 only for |t| < (N+tr)/2
    out = []
    for m in range(S):
        lo, hi = m * N - half + 1, m * N + half  # [lo, hi) in circular sample coordinates
        for sh in (-L, 0, L):
            if lo + sh < b and hi + sh > a:
                out.append(m)
                break
    return out


# ------------------------------------------------------------------ two-layer array
def two_layer(c_row_of_slices: np.ndarray, plan: Plan, L: int) -> List[np.ndarray]:
    """The paper's s = {s^0, s^1} (fig:slicqarray):
    s^{m mod 2}_k[((m-1) M_k/2 + n) mod (L M_k / 2N)] = c^m_k[n].
    Input: one signal's c[S][sum M]; output: per channel an array [2][L M_k / 2N]."""
    N2 = plan.sl_len
    S = c_row_of_slices.shape[0]
    off = offsets(plan)
    out = []
    for k, ch in enumerate(plan.stored):
        M = ch.M
        width = L * M // N2
        s = np.full((2, width), np.nan + 0j)
        for m in range(S):
            idx = np.mod((m - 1) * (M // 2) + np.arange(M), width)
            s[m % 2, idx] = c_row_of_slices[m, off[k]:off[k + 1]]
        out.append(s)
    return out


def from_two_layer(s: List[np.ndarray], plan: Plan, L: int) -> np.ndarray:
    """Partition s back into c^m (Alg. 4 lines P:338-340)."""
    S = 2 * L // plan.sl_len
    off = offsets(plan)
    c = np.zeros((S, plan.coeffs_per_slice), dtype=np.complex128)
    for k, ch in enumerate(plan.stored):
        M = ch.M
        width = s[k].shape[1]
        for m in range(S):
            idx = np.mod((m - 1) * (M // 2) + np.arange(M), width)
            c[m, off[k]:off[k + 1]] = s[k][m % 2, idx]
    return c


# ------------------------------------------------------------------ slice-range shards
def forward_range(x_local: np.ndarray, halo: int, slice0: int, nslices: int,
                  plan: Plan) -> np.ndarray:
    """Alg. 3 restricted to slices [slice0, slice0+nslices) of a long stream, from a
    local buffer whose index i holds global sample slice0*N - halo + i (the caller
    places the circularly wrapped samples, and zero padding).  Needs
    halo >= (N+tr)/2 - 1.  Returns c[nslices][sum M]."""
    N = plan.N
    assert halo >= (N + plan.tr) // 2 - 1
    out = np.zeros((nslices, plan.coeffs_per_slice), dtype=np.complex128)
    for i in range(nslices):
        m = slice0 + i
        j = np.arange(2 * N)
        li = (m - slice0) * N - N + j + halo  # local index of global (m-1)N + j
        v = np.zeros(2 * N)
        ok = (li >= 0) & (li < x_local.shape[0])
        v[ok] = x_local[li[ok]]
        v = v * plan.h0
        out[i] = concat(analysis_real(v, plan))
    return out


def inverse_range(c_local: np.ndarray, slice0: int, nslices: int, plan: Plan, halo: int):
    """Alg. 4 restricted to slices [slice0, slice0+nslices): returns
    (y_local over global samples [slice0 N, (slice0+nslices) N), left_spill over the
    `halo` samples [slice0 N - halo, slice0 N)).  The caller adds the right
    neighbour's spill to the tail of y_local."""
    N = plan.N
    y = np.zeros(nslices * N + halo, dtype=np.float64)  # index 0 <-> slice0 N - halo
    for i in range(nslices):
        m = slice0 + i
        fm = synthesis_real(split(c_local[i], plan), plan) * plan.h0dual
        li = (m - slice0) * N - N + np.arange(2 * N) + halo
        ok = (li >= 0) & (li < y.shape[0])
        assert np.all(fm[~ok] == 0)
        np.add.at(y, li[ok], fm[ok])
    return y[halo:], y[:halo]


# ------------------------------------------------------------------ complex input
# Alg. 3 / Alg. 4 for complex signals f in C^L (the paper's general setting, and its
# Set 1): every slice goes through the full 2K+2-channel CQ-NSGT_2N (Table 1 incl.
# the mirror channels K+2..2K+1).  Coefficient rows are [sum over all 2K+2 M_k] in
# Table-1 channel order (stored channels 0..K+1, then the mirrors of K..1).
from .nsgt import analysis as _analysis, synthesis as _synthesis  # noqa: E402


def offsets_full(plan: Plan) -> np.ndarray:
    return np.concatenate([[0], np.cumsum([c.M for c in plan.full])]).astype(np.int64)


def slice_frame_complex(x: np.ndarray, m: int, plan: Plan, L: int) -> np.ndarray:
    """f^m[j] = f[((m-1)N + j) mod L] h_0[j - N] for complex f."""
    N = plan.N
    idx = np.mod((m - 1) * N + np.arange(2 * N), L)
    v = np.zeros(2 * N, dtype=np.complex128)
    ok = idx < x.shape[0]
    v[ok] = x[idx[ok]]
    return v * plan.h0


def forward_complex(x: np.ndarray, plan: Plan) -> np.ndarray:
    """Alg. 3 for complex signals x[batch][n] -> c[batch][S][sum over 2K+2 channels M_k]."""
    x = np.atleast_2d(np.asarray(x, dtype=np.complex128))
    B, n = x.shape
    L = padded_length(n, plan.sl_len)
    S = 2 * L // plan.sl_len
    out = np.zeros((B, S, int(offsets_full(plan)[-1])), dtype=np.complex128)
    for b in range(B):
        for m in range(S):
            out[b, m] = concat(_analysis(slice_frame_complex(x[b], m, plan, L), plan.full,
                                         plan.sl_len))
    return out


def inverse_complex(c: np.ndarray, plan: Plan, n: int) -> np.ndarray:
    """Alg. 4 for complex signals: all 2K+2 channels through Alg. 2, dual window,
    overlap-add -> y[batch][n] complex."""
    c = np.asarray(c)
    if c.ndim == 2:
        c = c[None]
    B, S, _ = c.shape
    L = padded_length(n, plan.sl_len)
    N = plan.N
    off = offsets_full(plan)
    y = np.zeros((B, L), dtype=np.complex128)
    for b in range(B):
        for m in range(S):
            chans = [c[b, m, off[k]:off[k + 1]] for k in range(len(plan.full))]
            fm = _synthesis(chans, plan.full, plan.dual_full, plan.sl_len)
            pos = np.mod((m - 1) * N + np.arange(2 * N), L)
            np.add.at(y[b], pos, fm * plan.h0dual)
    return y[:, :n]
