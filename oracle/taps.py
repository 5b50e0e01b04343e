"""Oracle: exact tap-offset tables and angle assignment.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package.  It shares no code
with the CUDA path (paper_2309_15812_b200/).

What it computes:
  * Def. 1, Eq. "coordinate" and Appendix Eq. coordinate1d:
        oh_k = floor( -(k - pad) * sin(theta) ),   ow_k = floor( (k - pad) * cos(theta) )
    the floor of the EXACT real value (reading R3).
  * Direction groups: D angles i*180/D, channels split into D equal groups.
  * Bilinear discretisation: base corners + fractional parts of the real
    offsets (bilinear_exact / bilinear_table).

Exactness: the angle is a binary double, i.e. a rational number of degrees.  By
Niven's theorem sin(t deg) for rational t is rational only when it is 0, +-1/2 or
+-1 (t = 0, 30, 90, 150, 180, 210, 270, 330 mod 360), and likewise cos (t = 0, 60,
90, 120, 180, 240, 270, 300).  Those cases are evaluated in exact rational
arithmetic (fractions.Fraction).  Otherwise m*sin(t) (m != 0 integer) is
irrational, so it is never an integer, and its floor is evaluated with mpmath at
80 significant digits; the distance to the nearest integer is asserted to be far
above the evaluation error, so the floor is exact.
"""
from __future__ import annotations

from fractions import Fraction

import mpmath

_DPS = 80

# Niven's theorem tables (degrees mod 360 -> exact rational value)
_SIN_RATIONAL = {0: Fraction(0), 30: Fraction(1, 2), 90: Fraction(1), 150: Fraction(1, 2),
                 180: Fraction(0), 210: Fraction(-1, 2), 270: Fraction(-1), 330: Fraction(-1, 2)}
_COS_RATIONAL = {0: Fraction(1), 60: Fraction(1, 2), 90: Fraction(0), 120: Fraction(-1, 2),
                 180: Fraction(-1), 240: Fraction(-1, 2), 270: Fraction(0), 300: Fraction(1, 2)}


def _reduce_deg(theta_deg: float) -> Fraction:
    return Fraction(theta_deg) % 360


def _exact_value_times(m: Fraction, t: Fraction, fn: str):
    """m * fn(t degrees): an exact Fraction at the Niven angles, else an 80-digit mpf
    (irrational for m != 0)."""
    table = _SIN_RATIONAL if fn == "sin" else _COS_RATIONAL
    if m == 0:
        return Fraction(0)
    if t.denominator == 1 and int(t) in table:
        return m * table[int(t)]
    with mpmath.workdps(_DPS):
        tt = mpmath.mpf(t.numerator) / t.denominator
        rad = tt * mpmath.pi / 180
        mm = mpmath.mpf(m.numerator) / m.denominator
        return mm * (mpmath.sin(rad) if fn == "sin" else mpmath.cos(rad))


def _exact_floor_times(m, t: Fraction, fn: str) -> int:
    """floor(m * fn(t degrees)) exactly, fn in {"sin", "cos"}; m = k - pad is rational
    (pad may be any binary double, Eq. coordinate1d)."""
    m = Fraction(m)
    v = _exact_value_times(m, t, fn)
    if isinstance(v, Fraction):
        return v.numerator // v.denominator  # Fraction floor
    with mpmath.workdps(_DPS):
        f = int(mpmath.floor(v))
        dist = min(v - f, f + 1 - v)
        # irrational (Niven) => not an integer; must be resolvable at this precision
        assert dist > mpmath.mpf(10) ** (-(_DPS - 20)), (m, t, fn)
    return f


def taps_exact(K: int, pad, theta_deg: float):
    """Exact tap table for one angle: list of (oh_k, ow_k), k = 0..K-1.
    pad: an int or any float (taken as its exact binary value)."""
    t = _reduce_deg(theta_deg)
    out = []
    for k in range(K):
        m = k - Fraction(pad)
        oh = _exact_floor_times(-m, t, "sin")   # floor(-(k-pad) sin θ)
        ow = _exact_floor_times(m, t, "cos")    # floor( (k-pad) cos θ)
        out.append((oh, ow))
    return out


def bilinear_exact(K: int, pad, theta_deg: float):
    """Bilinear discretisation (Sec. "Discretization and Interpolation"): tap k
    samples x at the REAL offset of Eq. coordinate2d restricted to the 1D
    kernel (r = 0, s = k, pad_w = pad):  (u, v) = (-(k-pad) sin θ, (k-pad) cos θ).
    Returns per tap (h0, w0, a, b): the integer base corner h0 = floor(u), w0 = floor(v)
    (exact, = taps_exact) and the fractional parts a = u - h0, b = v - w0 in [0, 1)
    (exact at the Niven angles, else evaluated at 80 digits and rounded to f64).  The
    interpolated sample is (1-a)(1-b) x[h0][w0] + (1-a) b x[h0][w0+1] + a (1-b) x[h0+1][w0]
    + a b x[h0+1][w0+1] (reading R14)."""
    t = _reduce_deg(theta_deg)
    out = []
    for k in range(K):
        m = k - Fraction(pad)
        u = _exact_value_times(-m, t, "sin")
        v = _exact_value_times(m, t, "cos")
        h0 = _exact_floor_times(-m, t, "sin")
        w0 = _exact_floor_times(m, t, "cos")
        with mpmath.workdps(_DPS):
            a = float(u - h0) if isinstance(u, Fraction) else float(u - h0)
            b = float(v - w0) if isinstance(v, Fraction) else float(v - w0)
        out.append((h0, w0, a, b))
    return out


def bilinear_table(K: int, pad, angles_deg):
    """Per-channel bilinear tables: (h0[C][K], w0[C][K], a[C][K], b[C][K]) nested lists."""
    cache = {}
    h0, w0, fa, fb = [], [], [], []
    for ang in angles_deg:
        key = float(ang)
        if key not in cache:
            cache[key] = bilinear_exact(K, pad, key)
        rows = cache[key]
        h0.append([r[0] for r in rows])
        w0.append([r[1] for r in rows])
        fa.append([r[2] for r in rows])
        fb.append([r[3] for r in rows])
    return h0, w0, fa, fb


# Shear parameterisation (Appendix "Rotation vs Shearing").  The filter
# offset of tap k is sampled where the filter axis crosses integer columns,
# (delta_h, delta_w) = (-(k-pad) tan t, k-pad) (shear matrix S^x), or integer
# rows, ((k-pad), -(k-pad) cot t) (S^y); then floored as in Eq. coordinate1d.
# Readings (R13): the column form is used when |cos t| >= |sin t| (the axis
# is closer to horizontal), the row form otherwise; the offsets keep the direction of
# the rotation form (-sin t, cos t) -- i.e. offset = m * (-sin t, cos t) / max(|sin t|,
# |cos t|), m = k - pad -- so both forms agree with the rotation taps at 0 and 90 deg
# and tap k keeps its side of the centre.  P:432's worked example (t = -45 deg,
# pad = 0: offsets k(1, 1)) follows.
#
# Exactness: tan t for rational t (degrees) is rational only at t = 0, 45, 135 (mod
# 180) (Niven), where it is 0 or +-1; there the offset is evaluated exactly.  Otherwise
# m tan t (m != 0) is irrational and its floor is taken at 80 digits with the
# distance to the nearest integer asserted, as for the rotation form.
_TAN_RATIONAL = {0: Fraction(0), 45: Fraction(1), 135: Fraction(-1)}  # degrees mod 180


def _exact_floor_shear(m: int, t: Fraction, use_cols: bool, coord: str) -> int:
    """floor of one coordinate of m * (-sin t, cos t) / max(|sin t|, |cos t|)."""
    if m == 0:
        return 0
    u = t % 180
    sgn_cos = 1 if (t < 90 or t > 270) else (-1 if 90 < t < 270 else 0)
    sgn_sin = 1 if 0 < t < 180 else (-1 if t > 180 else 0)
    if use_cols:  # |cos| >= |sin|: delta_w = m sgn(cos t), delta_h = -m tan(t) sgn(cos t)
        if coord == "w":
            return m * sgn_cos
        if u.denominator == 1 and int(u) in _TAN_RATIONAL:
            v = -m * _TAN_RATIONAL[int(u)] * sgn_cos
            return v.numerator // v.denominator
        fn = lambda r: -m * mpmath.tan(r) * sgn_cos
    else:  # |sin| > |cos|: delta_h = -m sgn(sin t), delta_w = m cot(t) sgn(sin t)
        if coord == "h":
            return -m * sgn_sin
        if u == 90:
            return 0
        fn = lambda r: m * mpmath.cot(r) * sgn_sin
    with mpmath.workdps(_DPS):
        rad = mpmath.mpf(t.numerator) / t.denominator * mpmath.pi / 180
        v = fn(rad)
        f = int(mpmath.floor(v))
        dist = min(v - f, f + 1 - v)
        assert dist > mpmath.mpf(10) ** (-(_DPS - 20)), (m, t, coord)
    return f


def taps_exact_shear(K: int, pad: int, theta_deg: float):
    """Exact shear-form tap table for one angle: list of (oh_k, ow_k)."""
    t = _reduce_deg(theta_deg)
    u = t % 180
    use_cols = u <= 45 or u >= 135  # |cos t| >= |sin t|
    return [(_exact_floor_shear(k - pad, t, use_cols, "h"), _exact_floor_shear(k - pad, t, use_cols, "w"))
            for k in range(K)]


def taps_table(K: int, pad, angles_deg, mode: str = "rotation"):
    """Per-channel tables: (oh[C][K], ow[C][K]) as nested lists of int.  mode:
    "rotation" (Def. 1, the paper's default) or "shear" (Appendix)."""
    if mode not in ("rotation", "shear"):
        raise ValueError("mode must be 'rotation' or 'shear'")
    one = taps_exact if mode == "rotation" else taps_exact_shear
    cache = {}
    oh, ow = [], []
    for a in angles_deg:
        key = float(a)
        if key not in cache:
            cache[key] = one(K, pad, key)
        t = cache[key]
        oh.append([p[0] for p in t])
        ow.append([p[1] for p in t])
    return oh, ow


def direction_angles(D: int, C: int, assign: str = "contiguous", shift_deg: float = 0.0):
    """Angle per channel (degrees): D angles i*180/D, channels in D equal
    groups.  "contiguous": group of channel c is floor(c*D/C) (SPEC S:128 reading);
    "cycled": group is c mod D (BASELINE.json configs[1] reading).  The D=C case
    gives channel c the angle c*180/C under both readings.  shift_deg adds a
    layer-wise rotation ("alternating 90 deg"), reduced mod 180."""
    if D < 1 or C < 1 or (C % D != 0 and D != C):
        raise ValueError("D must divide C (or D == C)")
    out = []
    for c in range(C):
        g = (c * D) // C if assign == "contiguous" else c % D
        a = Fraction(g * 180, D) + Fraction(shift_deg)
        if shift_deg:
            a = a % 180
        out.append(float(a))
    return out
