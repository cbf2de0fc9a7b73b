"""Pins of the complex-input sliCQ oracle (oracle/slicq.py forward_complex / inverse_complex:
Alg. 3/4 over all 2K+2 channels of Table 1, the paper's general setting f in C^L):

  * perfect reconstruction of complex signals (Prop. 3)
  * every coefficient of one slice equals the explicit inner product <f^m, phi_{n,k}>
    (eq:CQ_coeff; oracle/direct.py), mirrors included
  * real input: the stored channels equal the real-input path and the mirror channels obey
    the Table-1 symmetry c_{n,2K+2-k} = e^{2 pi i 2N n/M_k} conj(c_{n,k}) (C15)
  * the plateau self-relations used by the GPU's complex path: DC real, Nyquist
    c = e^{2 pi i 2N n/M} conj(c) for real input
"""
import numpy as np
import pytest

from oracle import cqplan, direct
from oracle import slicq as osl
from oracle.nsgt import mirror_coeffs

SMALL = [(8000.0, 150.0, None, 6, 128, 16, 0), (8000.0, 150.0, None, 6, 128, 16, 1),
         (44100.0, 300.0, None, 4, 256, 32, 2), (16000.0, 100.0, 6000.0, 8, 160, 20, 0)]


def _cx(seed, B, n):
    r = np.random.default_rng(seed)
    return r.standard_normal((B, n)) + 1j * r.standard_normal((B, n))


@pytest.mark.parametrize("args", SMALL)
def test_complex_perfect_reconstruction(args):
    p = cqplan.make_plan(*args)
    for n in (p.sl_len, 3 * p.sl_len + 17, 5):
        x = _cx(n, 2, n)
        y = osl.inverse_complex(osl.forward_complex(x, p), p, n)
        assert np.abs(y - x).max() <= 1e-10 * np.abs(x).max()


def test_complex_coefficients_are_inner_products():
    p = cqplan.make_plan(*SMALL[0])
    x = _cx(1, 1, 3 * p.sl_len)
    c = osl.forward_complex(x, p)[0]
    L = osl.padded_length(x.shape[1], p.sl_len)
    off = osl.offsets_full(p)
    for m in (0, 2, c.shape[0] - 1):
        fm = osl.slice_frame_complex(x[0], m, p, L)
        ref = direct.coefficients(fm, p.full, p.sl_len)
        for k in range(len(p.full)):
            assert np.abs(c[m, off[k]:off[k + 1]] - ref[k]).max() <= 1e-10 * max(1.0, np.abs(ref[k]).max())


@pytest.mark.parametrize("args", SMALL[:3])
def test_real_input_mirror_relations(args):
    p = cqplan.make_plan(*args)
    x = np.random.default_rng(4).standard_normal((1, 2 * p.sl_len))
    c = osl.forward_complex(x, p)[0]
    cs = osl.forward(x, p)[0]
    C = p.coeffs_per_slice
    assert np.abs(c[:, :C] - cs).max() <= 1e-12 * np.abs(cs).max()
    off = osl.offsets(p)
    offf = osl.offsets_full(p)
    K = p.layout.K
    for m in range(c.shape[0]):
        stored = [cs[m, off[k]:off[k + 1]] for k in range(K + 2)]
        mir = mirror_coeffs(stored, p)
        for i, kk in enumerate(range(K + 2, 2 * K + 2)):
            assert np.abs(c[m, offf[kk]:offf[kk + 1]] - mir[i]).max() <= 1e-10 * np.abs(cs).max()
        # plateaus: DC real; Nyquist c = e^{2 pi i 2N n/M} conj(c)
        assert np.abs(stored[0].imag).max() <= 1e-10 * np.abs(cs).max()
        M = p.stored[K + 1].M
        ph = np.exp(2j * np.pi * p.sl_len * np.arange(M) / M)
        assert np.abs(stored[K + 1] - ph * np.conj(stored[K + 1])).max() <= 1e-10 * np.abs(cs).max()
