"""Pins for oracle/taps.py: the exact tap rule and angle groups.

Each pin is something other than the oracle itself: values printed in the paper /
SPEC, tables derived independently, symbolic floors (sympy),
closed forms and invariants stated in the paper.
"""
import math

import pytest
import sympy

from oracle import taps as T
from tests.golden_io import read_rows, read_tables


def test_spec_k3_tables():
    # SPEC.md S:104-106
    for th, tab in read_tables("taps_spec_k3.txt").items():
        assert T.taps_exact(3, 1, th) == tab, th


def test_paper_neg45_pad0():
    # theta=-45deg, pad=0 -> offsets k(sqrt2/2, sqrt2/2), floored
    rows = read_rows("taps_paper_neg45_pad0.txt")
    got = T.taps_exact(len(rows), 0, -45.0)
    assert got == [(int(oh), int(ow)) for _, oh, ow in rows]


def test_survey_k7_tables_and_hazard():
    # SURVEY.md Appendix A, incl. the 30 deg hazard where naive f64 floors are wrong
    for th, tab in read_tables("taps_survey_k7.txt").items():
        assert T.taps_exact(7, 3, th) == tab, th


def test_survey_k31_d8_tables():
    tabs = read_tables("taps_survey_k31_d8.txt")
    assert len(tabs) == 8
    distinct = []
    for th, tab in tabs.items():
        assert T.taps_exact(31, 15, th) == tab, th
        distinct.append(len(set(tab)))
    assert distinct == [31, 31, 23, 31, 31, 30, 22, 30]


@pytest.mark.parametrize("K", [3, 5, 7, 9])
def test_symbolic_floor_sympy(K):
    """Brute force with exact symbolic arithmetic: sympy floors of -(k-pad) sin(pi t/180)
    and (k-pad) cos(pi t/180) for integer degrees t in steps of 7.5 (covers the 30/60/90 family)."""
    pad = K // 2
    for i in range(0, 48):
        t = sympy.Rational(15, 2) * i
        ang = sympy.pi * t / 180
        s, c = sympy.sin(ang), sympy.cos(ang)
        want = [(int(sympy.floor(-(k - pad) * s)), int(sympy.floor((k - pad) * c))) for k in range(K)]
        assert T.taps_exact(K, pad, float(t)) == want, float(t)


@pytest.mark.parametrize("K", [3, 7, 15, 31, 63])
def test_invariants(K):
    pad = K // 2
    for t in [x * 0.5 for x in range(0, 720, 7)] + [0.0, 30.0, 60.0, 90.0, 120.0, 150.0, 22.5]:
        tab = T.taps_exact(K, pad, t)
        # origin of the convolution is angle independent
        assert tab[pad] == (0, 0)
        # offsets stay within the centred K x K window
        assert all(abs(a) <= pad and abs(b) <= pad for a, b in tab)
        # 180 deg reversal: taps(t+180)[k] == taps(t)[K-1-k]
        assert T.taps_exact(K, pad, t + 180.0) == tab[::-1]
    # closed forms at the axes
    assert T.taps_exact(K, pad, 0.0) == [(0, k - pad) for k in range(K)]
    assert T.taps_exact(K, pad, 90.0) == [(pad - k, 0) for k in range(K)]
    assert T.taps_exact(K, pad, 270.0) == [(k - pad, 0) for k in range(K)]


def test_naive_f64_hazard_documented():
    """Reading R3: naive f64 floors differ from the exact rule at 90 and 30 deg."""
    def naive(K, pad, t):
        r = math.radians(t)
        return [(math.floor(-(k - pad) * math.sin(r)), math.floor((k - pad) * math.cos(r))) for k in range(K)]
    assert naive(7, 3, 90.0) != T.taps_exact(7, 3, 90.0)
    assert naive(7, 3, 30.0) != T.taps_exact(7, 3, 30.0)


def test_direction_angles_paper_example():
    # D=4, C=512 -> 4 groups of 128 channels at 0, 45, 90, 135 deg
    a = T.direction_angles(4, 512, "contiguous")
    assert a[:128] == [0.0] * 128 and a[128:256] == [45.0] * 128
    assert a[256:384] == [90.0] * 128 and a[384:] == [135.0] * 128
    # SPEC S:131-133
    assert T.direction_angles(4, 8) == [0, 0, 45, 45, 90, 90, 135, 135]
    assert T.direction_angles(2, 4) == [0, 0, 90, 90]
    assert T.direction_angles(4, 4) == [0, 45, 90, 135]
    # BASELINE configs[1] "cycled" reading
    assert T.direction_angles(4, 8, "cycled") == [0, 45, 90, 135, 0, 45, 90, 135]
    # layer-wise rotation, SPEC S:137-139 ("alternating 90 deg", mod 180)
    assert T.direction_angles(4, 4, "contiguous", 90.0) == [90, 135, 0, 45]
    with pytest.raises(ValueError):
        T.direction_angles(3, 8)
