"""Mutation checks of the oracle's filter pins ("What's weak" 1): plausible
mistakes in oracle/cqplan.py's filter values must make a pin fail.  Each case patches the
oracle and runs the pins of tests/test_oracle_filters.py; at least one has to fail."""
import numpy as np
import pytest

from oracle import cqplan
import test_oracle_filters as pins


def _hann_cos(x):  # dropped square: H = cos(pi x)
    x = np.asarray(x, dtype=np.float64)
    return np.where(np.abs(x) <= 0.5, np.cos(np.pi * np.clip(x, -0.5, 0.5)), 0.0)


def _plateau_half(orig):  # g_0 = 1 - g_1 / 2
    def f(cq, Ls):
        (a, g0), (b, gn) = orig(cq, Ls)
        lo1, g1, _, _ = cq[0]
        j0 = np.arange(a, a + g0.shape[0])
        return (a, 1.0 - 0.5 * cqplan._eval_on(lo1, g1, np.abs(j0))), (b, gn)
    return f


def _plateau_nyq_sq(orig):  # Nyquist plateau squared (a plausible shape mix-up)
    def f(cq, Ls):
        (a, g0), (b, gn) = orig(cq, Ls)
        return (a, g0), (b, gn ** 2)
    return f


def _run_pins():
    failed = 0
    checks = [pins.test_hann_closed_form_points, pins.test_hann_half_period_partition_of_unity]
    checks += [lambda r=r: pins.test_frame_diagonal_range_matches_survey(*r) for r in pins._drows()]
    for c in checks:
        try:
            c()
        except AssertionError:
            failed += 1
    return failed


@pytest.mark.parametrize("name", ["hann_cos", "plateau_half", "plateau_nyq_sq"])
def test_mutation_is_caught(monkeypatch, name):
    if name == "hann_cos":
        monkeypatch.setattr(cqplan, "hann", _hann_cos)
        monkeypatch.setitem(cqplan.WINDOWS, "hann", _hann_cos)
    elif name == "plateau_half":
        monkeypatch.setattr(cqplan, "plateau_filters", _plateau_half(cqplan.plateau_filters))
    else:
        monkeypatch.setattr(cqplan, "plateau_filters", _plateau_nyq_sq(cqplan.plateau_filters))
    assert _run_pins() > 0


def test_unmutated_pins_pass():
    assert _run_pins() == 0
