"""C-ABI library checks that need no GPU: the library loads, exports every symbol
include/slicq.h declares, validates parameters, and its float64 host plan equals the
oracle's independently computed plan (plan parity, SURVEY §8(c) note)."""
import os
import re

import numpy as np
import pytest

from oracle import cqplan, slicq as oslicq
from synth.configs import CONFIGS, plan_args

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "slicq.h")


@pytest.fixture(scope="module")
def api():
    from paper_1210_0084_b200 import build
    build.build()
    from paper_1210_0084_b200 import api as _api
    return _api


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^SLICQ_API\s+[\w\s\*]*?\b(\w+)\(", txt, flags=re.M)))


def test_library_exports_every_declared_symbol(api):
    from paper_1210_0084_b200 import _lib
    L = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.SIGNATURES), "binding and header disagree"


def _plan_pair(api, args):
    lib_plan = api.Plan(*args, host_only=True)
    ref = cqplan.make_plan(*args)
    return lib_plan, ref


PLANS = [plan_args(CONFIGS[c]) for c in (1, 2, 3, 4, 5)] + [
    (44100.0, 65.4, 22050.0, 12, 16384, 2048, 1),
    (44100.0, 65.4, 22050.0, 12, 16384, 2048, 2),
    (8000.0, 150.0, 4000.0, 6, 128, 16, 0),
    (44100.0, 50.0, 20000.0, 48, 4096, 512, 0),
    (48000.0, 100.0, 30000.0, 24, 8192, 1024, 0),   # fmax above Nyquist: capped (C4)
    (22050.0, 30.0, 11025.0, 36, 32768, 4096, 0),
    (44100.0, 65.4, 22050.0, 12, 3 * 4096, 1000, 0),  # non power-of-two slice (host plan)
]


@pytest.mark.parametrize("args", PLANS)
def test_host_plan_parity_with_oracle(api, args):
    p, ref = _plan_pair(api, args)
    e = p.export()
    K2 = len(ref.stored)
    assert p.K == ref.layout.K and p.num_channels == K2
    assert np.array_equal(e["lo"], [c.lo for c in ref.stored])
    assert np.array_equal(e["len"], [c.L for c in ref.stored])
    assert np.array_equal(e["M"], [c.M for c in ref.stored])
    assert np.array_equal(e["off"], oslicq.offsets(ref))
    assert p.coeffs_per_slice == ref.coeffs_per_slice
    np.testing.assert_allclose(e["xi"], ref.layout.xi, rtol=1e-14)
    g_ref = np.concatenate([c.g for c in ref.stored])
    gd_ref = np.concatenate(ref.dual_stored)
    np.testing.assert_allclose(e["g"], g_ref, rtol=0, atol=1e-12)  # fp64 rounding order only
    np.testing.assert_allclose(e["gdual"], gd_ref, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(e["h0"], ref.h0, rtol=0, atol=1e-14)
    np.testing.assert_allclose(e["h0dual"], ref.h0dual, rtol=1e-13, atol=1e-14)
    assert p.halo == (ref.N + ref.tr) // 2


def test_queries(api):
    p = api.Plan(*plan_args(CONFIGS[1]), host_only=True)
    assert p.sl_len == 16384 and p.N == 8192
    for n, L in ((1, 16384), (16384, 16384), (16385, 32768), (65536, 65536), (441000, 442368)):
        assert p.padded_length(n) == L
        assert p.num_slices(n) == L // 8192
        assert oslicq.padded_length(n, 16384) == L
    assert p.workspace_bytes(8, 2) == 0  # layout depends on the device configuration


@pytest.mark.parametrize("bad", [
    (0.0, 65.4, 22050.0, 12, 16384, 2048, 0),
    (44100.0, -1.0, 22050.0, 12, 16384, 2048, 0),
    (44100.0, 30000.0, 32000.0, 12, 16384, 2048, 0),
    (44100.0, 65.4, 60.0, 12, 16384, 2048, 0),
    (44100.0, 65.4, 22050.0, 0, 16384, 2048, 0),
    (44100.0, 65.4, 22050.0, 12, 16386, 2048, 0),
    (44100.0, 65.4, 22050.0, 12, 7 * 2048, 2048, 0),
    (44100.0, 65.4, 22050.0, 12, 16384, 2047, 0),
    (44100.0, 65.4, 22050.0, 12, 16384, 8192, 0),
    (44100.0, 65.4, 22050.0, 12, 16384, 2048, 3),
])
def test_invalid_parameters_rejected(api, bad):
    from paper_1210_0084_b200._lib import SlicqError
    with pytest.raises(SlicqError) as ei:
        api.Plan(*bad, host_only=True)
    assert ei.value.code == -1  # SLICQ_EINVAL
    with pytest.raises(ValueError):
        cqplan.make_plan(*bad)


def test_hot_path_refuses_host_only_plan(api):
    import torch
    p = api.Plan(*plan_args(CONFIGS[1]), host_only=True)
    with pytest.raises((ValueError, RuntimeError)):
        p.forward(torch.zeros(1, 100))  # CPU tensor: there is no CPU path
