"""IEEE binary16 conversion, emulated with integer bit arithmetic.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Paper anchor: PAPER.md L262-269 (Sec. 3.2) -- "we also implemented the transfer
of parameters at half-precision while summing them at full precision".  The paper
does not state the conversion's rounding mode; reading Q6 fixes IEEE
round-to-nearest-even with gradual subnormals, and overflow (|x| >= 65520) to
+-inf.  SPEC.md L47-64 (numeric-core/to_half, from_half) gives worked values.

Functions
  rn16(x)   float32 array -> uint16 bit patterns   (round-to-nearest-even)
  widen(h)  uint16 bit patterns -> float32         (exact)
  overflow16(x) -> bool array: |x| rounds to +-inf (|x| >= 65520, finite x)

Pins (tests/test_oracle_fp16.py): golden values from SPEC L53-64 and the
binary16 format definition (tests/golden/rn16_values.txt); widen exhaustively
over all 65,536 patterns against the closed form (-1)^s 2^(e-15) (1+m/1024);
rn16 against an exact rational (fractions.Fraction) rounding on every fp32
exponent with random and tie mantissas, against CPython's struct 'e' codec, and
(opt-in, TM_EXHAUSTIVE=1) against numpy astype on all 2^32 inputs.
"""

import numpy as np

_U32 = np.uint32


def rn16(x):
    """Round float32 values to IEEE binary16, nearest-even.  Returns uint16 bits.

    Step by step (binary16: 1 sign, 5 exponent bits bias 15, 10 fraction bits):
      1. split the fp32 pattern into sign, biased exponent E (bias 127), fraction;
      2. NaN -> quiet NaN 0x7E00 (payload not preserved; outside parity, Q8),
         +-inf -> +-inf;
      3. half exponent e = E - 127 + 15.  If e >= 1 the result is normal: drop
         13 fraction bits, round half to even, let a carry ripple into the
         exponent (e = 31 after rounding is infinity, which is IEEE overflow);
      4. if e <= 0 the result is subnormal (unit 2^-24): the 24-bit significand
         (implicit 1 included) is shifted right by 126 - E, rounded half to even;
         a carry into bit 10 yields the smallest normal, as IEEE requires;
      5. fp32 subnormal inputs are below 2^-126 and round to signed zero.
    """
    x = np.ascontiguousarray(x, dtype=np.float32)
    b = x.view(_U32)
    sign = ((b >> _U32(16)) & _U32(0x8000)).astype(_U32)
    E = ((b >> _U32(23)) & _U32(0xFF)).astype(np.int64)
    frac = (b & _U32(0x7FFFFF)).astype(np.int64)

    out = np.zeros(x.shape, dtype=np.int64)

    # (3) normal half results: E >= 113  <=>  e >= 1.  E >= 143 overflows.
    e = E - 112
    normal = (E >= 113) & (E < 143)
    keep = frac >> 13
    rem = frac & 0x1FFF
    up = (rem > 0x1000) | ((rem == 0x1000) & ((keep & 1) == 1))
    out = np.where(normal, (e << 10) + keep + up.astype(np.int64), out)

    # overflow (finite fp32 with |x| >= 2^16) -> inf
    big = (E >= 143) & (E < 255)
    out = np.where(big, 0x7C00, out)

    # (4) subnormal half results: 1 <= E <= 112 (fp32 normals below 2^-14)
    sub = (E >= 1) & (E <= 112)
    sig = frac | 0x800000
    shift = np.minimum(126 - E, 40)  # >= 14 here; >= 25 always rounds to 0
    shift_c = np.where(sub, shift, 1)
    q = sig >> shift_c
    rem_s = sig & ((np.int64(1) << shift_c) - 1)
    half = np.int64(1) << (shift_c - 1)
    up_s = (rem_s > half) | ((rem_s == half) & ((q & 1) == 1))
    out = np.where(sub, q + up_s.astype(np.int64), out)

    # (5) E == 0: zero or fp32 subnormal -> signed zero (already 0)
    # (2) specials
    inf_in = (E == 255) & (frac == 0)
    nan_in = (E == 255) & (frac != 0)
    out = np.where(inf_in, 0x7C00, out)
    out = np.where(nan_in, 0x7E00, out)

    return (out.astype(_U32) | sign).astype(np.uint16)


def widen(h):
    """Exact binary16 -> float32 (every binary16 value is an fp32 value).

    normal   (1 <= e <= 30): fp32 exponent e + 112, fraction m << 13
    subnormal(e = 0, m > 0): value m * 2^-24; normalise at the leading bit p of m:
                             fp32 exponent p + 103, fraction (m << (23 - p)) & 0x7FFFFF
    zero, inf, NaN map to the same class with the sign kept.
    """
    h = np.ascontiguousarray(h, dtype=np.uint16).astype(np.int64)
    sign = (h & 0x8000) << 16
    e = (h >> 10) & 0x1F
    m = h & 0x3FF

    bits = np.where((e >= 1) & (e <= 30), ((e + 112) << 23) | (m << 13), 0)
    bits = np.where(e == 31, 0x7F800000 | (m << 13), bits)

    sub = (e == 0) & (m != 0)
    # leading-bit position p of m in [0, 9]
    p = np.zeros_like(m)
    for bit in range(10):
        p = np.where((m >> bit) & 1 == 1, bit, p)
    sub_bits = ((p + 103) << 23) | ((m << (23 - p)) & 0x7FFFFF)
    bits = np.where(sub, sub_bits, bits)

    bits = (bits | sign).astype(np.uint32)
    return bits.view(np.float32)


def overflow16(x):
    """True where a finite fp32 value rounds to +-inf in binary16 (|x| >= 65520).

    SPEC L49-51 (to_half errors: OverflowToInfinity).  65520 = 65504 + half an
    ulp(2^15) = (2 - 2^-11) * 2^15 is the RNE tie that rounds up to infinity."""
    x = np.asarray(x, dtype=np.float32)
    return np.isfinite(x) & (np.abs(x) >= np.float32(65520.0))
