"""ORACLE (test infrastructure only) — coefficients as explicit inner products.

eq:CQ_coeff: c_{n,k} = <f, phi_{n,k}> with the time-domain atom
phi_{n,k} = T_{n a_k} g_k-check.  With the C1 scaling of Alg. 1, on a
length-Ls frame (a_k = Ls/M_k):

    phi_{n,k}[l] = M_k^{-1/2} * sum_{j in J_k} g_k[j] exp(2 pi i j (l - n Ls/M_k) / Ls)

and c_{n,k} = sum_l f[l] conj(phi_{n,k}[l]).  This is an O(Ls * sum_k L_k * M_k)
double sum with no FFT, no folding and no periodization: it pins the scale, the
phase convention (C6) and the unwrapped folding (C5) of the FFT path.
Only for tiny Ls (<= 512).
"""
from __future__ import annotations

from typing import List, Sequence

import numpy as np

from .cqplan import Channel


def atom(c: Channel, n: int, Ls: int) -> np.ndarray:
    l = np.arange(Ls, dtype=np.float64)
    j = c.bins.astype(np.float64)
    ph = 2j * np.pi * np.outer(l - n * Ls / c.M, j) / Ls     # [l][j]
    return (np.exp(ph) @ c.g) / np.sqrt(c.M)


def coefficients(f: np.ndarray, channels: Sequence[Channel], Ls: int) -> List[np.ndarray]:
    f = np.asarray(f, dtype=np.complex128)
    out = []
    for c in channels:
        out.append(np.array([np.sum(f * np.conj(atom(c, n, Ls))) for n in range(c.M)]))
    return out


def frame_operator(channels: Sequence[Channel], Ls: int) -> np.ndarray:
    """Brute-force S = sum_{n,k} phi_{n,k} phi_{n,k}^H as an Ls x Ls matrix (eq:frameop)."""
    S = np.zeros((Ls, Ls), dtype=np.complex128)
    for c in channels:
        for n in range(c.M):
            a = atom(c, n, Ls)
            S += np.outer(a, np.conj(a))
    return S


def analysis_matrix(channels: Sequence[Channel], Ls: int) -> np.ndarray:
    """Rows phi_{n,k}^H, so that (A f) stacks all coefficients (channel-major)."""
    rows = []
    for c in channels:
        for n in range(c.M):
            rows.append(np.conj(atom(c, n, Ls)))
    return np.array(rows)
