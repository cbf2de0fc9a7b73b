"""Pins for the oracle's filter values (oracle/cqplan.py hann, cq_filter, plateau_filters).

Runs without a GPU.  These pin the VALUES of g_k and the plateaus g_0, g_{K+1}
(Table 1 rows k = 0 and K+1), which every GPU parity claim inherits:
  * H = cos^2(pi x) (reading C7) at closed-form points and by its half-period partition of
    unity -- a property of the Hann window, not a re-typed formula;
  * the frame diagonal's range per config against the survey's independent values
    (tests/golden/frame_diagonal.txt);
  * the plateaus reach 1 exactly where no CQ filter reaches ("plateau functions
    centered at 0 and Nyquist").
Mutations these catch (checked when written): H = cos(pi x) (H(1/4) = 0.707, cfg1 D range
[0.33, 1.42]) and g_0 = 1 - g_1 / 2 (cfg1 max D 1.17).
"""
import math
import os

import numpy as np
import pytest

from oracle import cqplan
from synth.configs import CONFIGS, plan_args

GOLD = os.path.join(os.path.dirname(__file__), "golden", "frame_diagonal.txt")


def _drows():
    out = []
    for line in open(GOLD):
        f = line.split()
        if f and f[0] == "D":
            out.append((int(f[1]), float(f[2]), float(f[3])))
    return out


def test_hann_closed_form_points():
    # H(0) = 1, H(+-1/4) = cos^2(pi/4) = 1/2, H(+-1/3) = cos^2(pi/3) = 1/4, H(+-1/2) = 0,
    # H = 0 outside [-1/2, 1/2]  (reading C7 of P:262)
    x = np.array([0.0, 0.25, -0.25, 1 / 3, -1 / 3, 0.5, -0.5, 0.6, -0.75, 3.0])
    want = np.array([1.0, 0.5, 0.5, 0.25, 0.25, 0.0, 0.0, 0.0, 0.0, 0.0])
    assert np.max(np.abs(cqplan.hann(x) - want)) < 1e-15


def test_hann_half_period_partition_of_unity():
    # cos^2(pi x) + cos^2(pi (x - 1/2)) = cos^2 + sin^2 = 1 on [0, 1/2]: the property that makes
    # 50 %-overlapping Hann filters a near-tight bank (P:135 footnote, north_star)
    x = np.linspace(0.0, 0.5, 1001)
    s = cqplan.hann(x) + cqplan.hann(x - 0.5)
    assert np.max(np.abs(s - 1.0)) < 1e-15
    # symmetric and monotone on [0, 1/2]
    assert np.array_equal(cqplan.hann(x), cqplan.hann(-x))
    assert np.all(np.diff(cqplan.hann(x)) <= 0)


@pytest.mark.parametrize("cfg,dmin,dmax", _drows())
def test_frame_diagonal_range_matches_survey(cfg, dmin, dmax):
    # D = sum_k |g_k|^2 over all 2K+2 channels (C16) against the survey's values
    p = cqplan.make_plan(*plan_args(CONFIGS[cfg]))
    assert abs(float(p.D.min()) - dmin) < 0.006
    assert abs(float(p.D.max()) - dmax) < 0.006


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_plateaus_reach_one_where_no_cq_filter_reaches(cfg):
    # the plateaus are 1 wherever no CQ filter (or its mirror) reaches -- at DC they are
    # "centered at 0" with value 1 (C8) -- and never exceed 1 (a partition with the
    # neighbouring CQ filter, not an extra gain)
    p = cqplan.make_plan(*plan_args(CONFIGS[cfg]))
    N2 = 2 * p.N
    dc, nyq = p.stored[0], p.stored[-1]
    c1, cK = p.stored[1], p.stored[-2]

    def touched(ch, j):
        return any(ch.lo <= jj < ch.lo + ch.L for jj in (j, -j, j + N2, j - N2, N2 - j))

    assert dc.g[-dc.lo] == 1.0  # j = 0
    assert dc.g.max() <= 1.0 and nyq.g.max() <= 1.0
    for plate, nb in ((dc, c1), (nyq, cK)):
        free = [j for j in range(plate.lo, plate.lo + plate.L) if not touched(nb, j)]
        assert free or plate is nyq  # (cfg1: the top CQ filter's mirror covers the plateau)
        for j in free:
            assert plate.g[j - plate.lo] == 1.0
