"""Exact rational restatement of the canonical FP32 distance (test helper).

Used to pin the oracle's arithmetic from outside: every FP32 operation is done
in exact rational arithmetic and rounded to nearest-even float32 by hand, so a
wrong operation order, a missing FMA, or a wrong wrap shows up as a bit
difference. Not shared with either implementation.
"""
from fractions import Fraction

import numpy as np


def rn32(x: Fraction) -> Fraction:
    """Round a rational to the nearest float32 (ties to even), subnormals honoured."""
    if x == 0:
        return Fraction(0)
    sign = -1 if x < 0 else 1
    a = -x if x < 0 else x
    # exponent e with 2^e <= a < 2^(e+1)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    elif Fraction(2) ** (e + 1) <= a:
        e += 1
    q = max(e, -126) - 23  # ulp exponent (subnormal ulp = 2^-149)
    m = a / (Fraction(2) ** q)
    fl = m.numerator // m.denominator
    rem = m - fl
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1):
        fl += 1
    return sign * Fraction(fl) * (Fraction(2) ** q)


def f(v) -> Fraction:
    return Fraction(float(np.float32(v)))


def canon_d2_exact(q, s, box=None) -> Fraction:
    t = []
    for d in range(3):
        td = rn32(f(q[d]) - f(s[d]))
        if box is not None:
            L = f(box[d] if np.ndim(box) else box)
            h = rn32(L / 2)
            if td >= h:
                td = rn32(td - L)
            elif td < -h:
                td = rn32(td + L)
        t.append(td)
    xx = rn32(t[0] * t[0])
    yy = rn32(t[1] * t[1] + xx)
    return rn32(t[2] * t[2] + yy)


def to_f32(x: Fraction) -> np.float32:
    return np.float32(float(x))


def brute_exact(pos, k, box=None, queries=None):
    """Pure-Python definition on tiny inputs: rows of (j, d2) sorted by (d2, j).
    queries=None: self-query; else row i answers queries[i] against the sources pos."""
    n = len(pos)
    qs = pos if queries is None else queries
    rows = []
    for i in range(len(qs)):
        cand = sorted((canon_d2_exact(qs[i], pos[j], box), j) for j in range(n))
        rows.append([(j, to_f32(d)) for d, j in cand[:k]])
    return rows
