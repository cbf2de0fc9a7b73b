"""Seeded synthetic input generators (SURVEY.md §8(d) "Synthetic inputs").

This module holds no transform arithmetic: it only draws audio-shaped test
signals.  Both the CUDA path (tests, bench) and the oracle tests take their
inputs from here, so the two sides see the *same* fp32 values (SURVEY §8(c)
C18: generated in float64, cast to float32 once).

The paper says timing "does not depend on signal content" and used random
signals; its music Set 2 and the Glockenspiel recording are not
available, so these generators stand in for them with audio-like structure.

Every generator uses numpy ``Generator(PCG64(seed))`` and draws its random
numbers in a fixed, documented order.
"""
from __future__ import annotations

import math

import numpy as np

from .configs import CONFIGS, SlicqConfig


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def cfg1_signal(c: SlicqConfig) -> np.ndarray:
    """sigma=0.1 Gaussian noise + 0.5*sin(2*pi*f*t/fs), f in {220, 1000, 5000} Hz, phase 0."""
    rng = _rng(c.seed)
    t = np.arange(c.n, dtype=np.float64) / c.fs
    x = 0.1 * rng.standard_normal(c.n)
    for f in (220.0, 1000.0, 5000.0):
        x += 0.5 * np.sin(2 * np.pi * f * t)
    return x.astype(np.float32)[None, :]


def cfg2_signal(c: SlicqConfig) -> np.ndarray:
    """Linear chirp 50 Hz -> 20 kHz over 10 s, + 20 consecutive 0.5 s harmonic tones
    (f0 ~ U(80, 800), partials p=1..10 with amplitude 0.25/p, random phases,
    partials >= fs/2 dropped), + sigma=0.01 noise.
    Draw order: 20 f0's, then 20x10 phases, then the noise."""
    rng = _rng(c.seed)
    n, fs = c.n, c.fs
    t = np.arange(n, dtype=np.float64) / fs
    T = n / fs
    x = 0.5 * np.sin(2 * np.pi * (50.0 * t + (20000.0 - 50.0) * t * t / (2.0 * T)))
    f0s = rng.uniform(80.0, 800.0, size=20)
    phases = rng.uniform(0.0, 2 * np.pi, size=(20, 10))
    seg = int(round(0.5 * fs))
    for i in range(20):
        a, b = i * seg, min(n, (i + 1) * seg)
        if a >= n:
            break
        tt = t[a:b]
        for p in range(1, 11):
            f = p * f0s[i]
            if f >= fs / 2:
                continue
            x[a:b] += (0.25 / p) * np.sin(2 * np.pi * f * tt + phases[i, p - 1])
    x += 0.01 * rng.standard_normal(n)
    return x.astype(np.float32)[None, :]


def pink_noise(rng: np.random.Generator, n: int) -> np.ndarray:
    """White Gaussian -> rFFT -> bin j scaled by j^-1/2 (DC = 0) -> irFFT -> unit RMS."""
    w = rng.standard_normal(n)
    W = np.fft.rfft(w)
    j = np.arange(W.shape[0], dtype=np.float64)
    scale = np.zeros_like(j)
    scale[1:] = j[1:] ** -0.5
    p = np.fft.irfft(W * scale, n)
    return p / np.sqrt(np.mean(p * p))


def cfg3_signal(c: SlicqConfig, batch: int | None = None) -> np.ndarray:
    """64 stereo signals = 128 i.i.d. pink-noise channels of 2^20 samples."""
    rng = _rng(c.seed)
    b = c.batch if batch is None else batch
    out = np.empty((b, c.n), dtype=np.float32)
    for i in range(b):
        out[i] = pink_noise(rng, c.n).astype(np.float32)
    return out


def cfg4_signal(c: SlicqConfig, n: int | None = None) -> np.ndarray:
    """One hour at 48 kHz: consecutive notes, duration ~ U(0.1, 1.0) s, MIDI pitch
    ~ U{28..100}, f0 = 440*2^((p-69)/12); each note sum_{q=1..8} (1/q) sin(2 pi q f0 t)
    (partials >= fs/2 dropped) times 0.5*exp(-t/tau), tau = duration/3; plus
    sigma=0.01 noise.  Draw order: all (duration, pitch) pairs, then the noise in
    chunks of 2^24 samples.  ``n`` truncates (the prefix is identical)."""
    rng = _rng(c.seed)
    n_full = c.n
    n = n_full if n is None else n
    fs = c.fs
    # Note parameters for the FULL stream are drawn first so that prefixes agree.
    durs, pitches = [], []
    total = 0
    while total < n_full:
        d = rng.uniform(0.1, 1.0)
        p = int(rng.integers(28, 101))
        ns = max(1, int(round(d * fs)))
        durs.append((d, ns))
        pitches.append(p)
        total += ns
    # noise, added in float64 chunk by chunk, then a single cast to fp32
    CH = 1 << 24
    out = np.empty(n, dtype=np.float32)
    note_starts = np.cumsum([0] + [ns for _, ns in durs])
    k = 0
    for a in range(0, n_full, CH):
        b = min(n_full, a + CH)
        if a >= n:
            break
        noise = 0.01 * rng.standard_normal(b - a)
        bb = min(b, n)
        seg = np.zeros(bb - a, dtype=np.float64)
        while k < len(durs) and note_starts[k + 1] <= a:
            k += 1
        kk = k
        while kk < len(durs) and note_starts[kk] < bb:
            s0 = note_starts[kk]
            d, ns = durs[kk]
            lo, hi = max(a, s0), min(bb, s0 + ns)
            tt = (np.arange(lo, hi, dtype=np.float64) - s0) / fs
            f0 = 440.0 * 2.0 ** ((pitches[kk] - 69) / 12.0)
            ph = 2 * np.pi * f0 * tt
            # sin(q*ph), q = 1..8, by the Chebyshev recurrence
            # sin((q+1)x) = 2 cos(x) sin(qx) - sin((q-1)x)  (fp64; q <= 8)
            s1 = np.sin(ph)
            c2 = 2.0 * np.cos(ph)
            s = s1.copy()
            sq_prev, sq = np.zeros_like(s1), s1
            for q in range(2, 9):
                if q * f0 >= fs / 2:
                    break
                sq_prev, sq = sq, c2 * sq - sq_prev
                s += sq / q
            seg[lo - a:hi - a] += s * 0.5 * np.exp(-tt / (d / 3.0))
            kk += 1
        seg += noise[:bb - a]
        out[a:bb] = seg.astype(np.float32)
    return out[None, :]


def cfg5_signal(c: SlicqConfig, batch: int | None = None, n: int | None = None) -> np.ndarray:
    """16 signals of 2^22 samples: 64 sinusoids per signal, f = exp(U(ln 27.5, ln 20000)),
    phase U(0, 2 pi), amplitude 1/8 each; plus sigma=0.05 white noise.
    Draw order per signal: 64 frequencies, 64 phases, then the noise."""
    rng = _rng(c.seed)
    b = c.batch if batch is None else batch
    n_full = c.n
    n = n_full if n is None else n
    out = np.empty((b, n), dtype=np.float32)
    blk = 4096  # angle addition per block: sin(w(t0+u)+p) = sin(wt0+p)cos(wu) + cos(wt0+p)sin(wu)
    nb = -(-n // blk)
    u = np.arange(blk, dtype=np.float64) / c.fs
    t0 = np.arange(nb, dtype=np.float64) * (blk / c.fs)
    for i in range(b):
        f = np.exp(rng.uniform(math.log(27.5), math.log(20000.0), size=64))
        ph = rng.uniform(0.0, 2 * np.pi, size=64)
        noise = 0.05 * rng.standard_normal(n_full)[:n]
        w = 2 * np.pi * f
        arg0 = np.outer(t0, w) + ph                      # [nb][64] phase at each block start
        cu, su = np.cos(np.outer(w, u)), np.sin(np.outer(w, u))  # [64][blk]
        x = (np.sin(arg0) @ cu + np.cos(arg0) @ su).reshape(-1)[:n]
        out[i] = (noise + 0.125 * x).astype(np.float32)
    return out


_GEN = {1: cfg1_signal, 2: cfg2_signal, 3: cfg3_signal, 4: cfg4_signal, 5: cfg5_signal}


def make_signal(cfg: int, **kw) -> np.ndarray:
    """fp32 array [batch][n] for BASELINE config ``cfg`` (1..5)."""
    return _GEN[cfg](CONFIGS[cfg], **kw)


def random_signal(seed: int, batch: int, n: int, scale: float = 1.0) -> np.ndarray:
    """Generic seeded Gaussian fp32 test input (edge cases, small parity shapes)."""
    rng = _rng(seed)
    return (scale * rng.standard_normal((batch, n))).astype(np.float32)
