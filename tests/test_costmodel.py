"""Cost model (costmodel.py restated): profile parsing / interpolation and the analytic
speedup, checked against the reference's own formulas on its illustrative profile."""

from __future__ import annotations

from fractions import Fraction

import pytest

from paper_2410_11305_b200 import costmodel as CM

PROFILE = """
draft batch=1 cost=0.3
draft batch=16 cost=0.32
verify batch=1 n=1 cost=1.0
verify batch=1 n=4 cost=1.15
verify batch=16 n=1 cost=1.0
verify batch=16 n=2 cost=1.05
verify batch=16 n=4 cost=1.15
"""


def test_parse_format_interpolate():
    p = CM.parse_profile(PROFILE)
    assert CM.parse_profile(CM.format_profile(p)).draft == p.draft
    assert float(p.draft_cost(8)) == pytest.approx(0.3 + 0.02 * 7 / 15)
    assert float(p.verify_cost(16, 3)) == pytest.approx(1.10)
    assert p.base_cost(1) == 1
    with pytest.raises(CM.ProfileError):
        p.draft_cost(17)
    with pytest.raises(CM.ProfileError):
        CM.parse_profile("verify batch=1 n=2 cost=1.0")     # no n=1 baseline


def test_analytic_speedup_formula():
    p = CM.parse_profile(PROFILE)
    acc = CM.AcceptanceModel.from_trace([3, 3, 1, 0], 3)
    r = CM.analytic_speedup(p, acc, 3, 1)
    tpc = Fraction(7, 4) + 1
    assert r.tokens_per_cycle == pytest.approx(float(tpc))
    assert r.speedup == pytest.approx(float(tpc) / (3 * 0.3 + 1.15))
    g = CM.geometric_acceptance(0.5, 3)
    assert float(g.expected_accept_len()) == pytest.approx(0.5 + 0.25 + 0.125)
