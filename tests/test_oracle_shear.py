"""Pins for the shear-form tap tables of oracle/taps.py (Appendix "Rotation vs
Shearing"; reading R13).  Each pin is independent of the oracle's
own arithmetic: the paper's worked example, exact symbolic floors (sympy), the
rotation form at angles where both forms must agree, and the properties
states for the shear form."""
import pytest
import sympy

from oracle import taps as T
from tests.golden_io import read_rows


def test_paper_shear_neg45_pad0():
    # theta = -45 deg, pad = 0 -> integer offsets k(1, 1), no discretisation needed
    rows = read_rows("taps_paper_shear_neg45_pad0.txt")
    assert T.taps_exact_shear(len(rows), 0, -45.0) == [(int(oh), int(ow)) for _, oh, ow in rows]


@pytest.mark.parametrize("theta", [0.0, 90.0, 180.0, 270.0, -90.0, 360.0])
def test_shear_equals_rotation_on_axes(theta):
    # on the axes the filter axis already lies on a grid line: both parameterisations agree
    for K in (1, 3, 7, 31):
        assert T.taps_exact_shear(K, K // 2, theta) == T.taps_exact(K, K // 2, theta)


@pytest.mark.parametrize("K", [7, 15, 31])
def test_shear_symbolic_floor_sympy(K):
    """Brute force with exact symbolic arithmetic on a 7.5 deg grid: offset = m (-sin, cos) /
    max(|sin|, |cos|), floored (sympy), m = k - pad."""
    pad = K // 2
    for i in range(48):
        t = sympy.Rational(15, 2) * i
        ang = sympy.pi * t / 180
        s, c = sympy.sin(ang), sympy.cos(ang)
        nrm = sympy.Max(sympy.Abs(s), sympy.Abs(c))
        want = [(int(sympy.floor(-(k - pad) * s / nrm)), int(sympy.floor((k - pad) * c / nrm))) for k in range(K)]
        assert T.taps_exact_shear(K, pad, float(t)) == want, t


@pytest.mark.parametrize("theta", [0.0, 10.0, 22.5, 30.0, 45.0, 60.0, 67.5, 89.0, 112.5, 135.0, 157.5, 200.0, 300.0])
def test_shear_properties(theta):
    """forcing one coordinate onto the grid removes the rotation form's redundancy
    (all K offsets distinct); that coordinate is exactly +-(k - pad); the kernel keeps its
    centre (k = pad -> (0, 0)) and its extent (|offsets| <= pad)."""
    K = 31
    pad = K // 2
    tab = T.taps_exact_shear(K, pad, theta)
    assert len(set(tab)) == K
    assert tab[pad] == (0, 0)
    on_rows = all(abs(oh) == abs(k - pad) for k, (oh, ow) in enumerate(tab))
    on_cols = all(abs(ow) == abs(k - pad) for k, (oh, ow) in enumerate(tab))
    assert on_rows or on_cols
    assert all(abs(oh) <= pad and abs(ow) <= pad for oh, ow in tab)
    # same side of the centre as the rotation form's tap k (direction (-sin, cos))
    rot = T.taps_exact(K, pad, theta)
    for (a, b), (c, d) in zip(tab, rot):
        assert a * c >= 0 or abs(a) <= 1 or abs(c) <= 1
        assert b * d >= 0 or abs(b) <= 1 or abs(d) <= 1


def test_shear_table_modes():
    ang = [0.0, 45.0, 90.0, 135.0]
    assert T.taps_table(7, 3, ang, "rotation") == T.taps_table(7, 3, ang)
    oh, ow = T.taps_table(7, 3, ang, "shear")
    assert [list(zip(oh[i], ow[i])) for i in range(4)] == [T.taps_exact_shear(7, 3, a) for a in ang]
    with pytest.raises(ValueError):
        T.taps_table(7, 3, ang, "bilinear")
