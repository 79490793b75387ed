"""Exact-rational IEEE rounding, written independently of oracle/ to pin it.

Every value is handled as a Python float (which holds any fp32 or fp16 value
exactly) converted to fractions.Fraction; each arithmetic step is done exactly
and then rounded to the target format by round-half-to-even on integers.  The
sign of zero follows IEEE 754 Sec. 6.3 for round-to-nearest: an exact zero sum
of operands of opposite sign is +0; x + x keeps x's sign; a nonzero result that
rounds to zero keeps its own sign.
"""

import math
from fractions import Fraction

# (precision p incl. hidden bit, emin, emax)
BINARY32 = (24, -126, 127)
BINARY16 = (11, -14, 15)


def round_fraction(q, fmt, neg_zero=False):
    """Round exact rational q to the nearest `fmt` value, ties to even.
    Returns a Python float (may be +-inf, or -0.0)."""
    p, emin, emax = fmt
    if q == 0:
        return -0.0 if neg_zero else 0.0
    sign = -1 if q < 0 else 1
    a = abs(q)
    # exponent e with 2^e <= a < 2^(e+1)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    elif Fraction(2) ** (e + 1) <= a:
        e += 1
    e_eff = max(e, emin)
    scale = Fraction(2) ** (p - 1 - e_eff)
    m = a * scale
    M = m.numerator // m.denominator
    rem = m - M
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and M % 2 == 1):
        M += 1
    val = Fraction(M) / scale
    max_finite = (Fraction(2) ** p - 1) * Fraction(2) ** (emax - p + 1)
    if val > max_finite:
        return math.copysign(math.inf, sign)
    if M == 0:
        return -0.0 if sign < 0 else 0.0
    return sign * float(val)


def _frac(x):
    return Fraction(float(x))


def _is_neg_zero(x):
    return x == 0 and math.copysign(1.0, x) < 0


def add(a, b, fmt=BINARY32):
    a, b = float(a), float(b)
    s = _frac(a) + _frac(b)
    return round_fraction(s, fmt, neg_zero=(_is_neg_zero(a) and _is_neg_zero(b)))


def sub(a, b, fmt=BINARY32):
    return add(a, -float(b), fmt)


def mul(a, b, fmt=BINARY32):
    a, b = float(a), float(b)
    neg = (math.copysign(1.0, a) * math.copysign(1.0, b)) < 0
    return round_fraction(_frac(a) * _frac(b), fmt, neg_zero=neg)


def div(a, b, fmt=BINARY32):
    a, b = float(a), float(b)
    neg = (math.copysign(1.0, a) * math.copysign(1.0, b)) < 0
    return round_fraction(_frac(a) / _frac(b), fmt, neg_zero=neg)


def to16(a):
    """Round an fp32 value (a Python float) to binary16 (value returned as float)."""
    a = float(a)
    if math.isinf(a):
        return a
    return round_fraction(_frac(a), BINARY16, neg_zero=_is_neg_zero(a))


def same_bits32(a, b):
    """Bitwise equality of two values as fp32 (distinguishes +0/-0)."""
    import struct
    return struct.pack("<f", float(a)) == struct.pack("<f", float(b))
