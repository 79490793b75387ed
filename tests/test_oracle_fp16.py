"""Pins for oracle/fp16.py against things other than itself (CPU only)."""

import math
import os
import struct

import numpy as np
import pytest

import exact
from oracle.fp16 import overflow16, rn16, widen

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "rn16_values.txt")


def _golden_rows():
    rows = []
    with open(GOLDEN) as f:
        for line in f:
            if not line.strip() or line.startswith("#"):
                continue
            parts = line.split()
            rows.append((int(parts[0], 16), int(parts[1], 16), float(parts[2]), " ".join(parts[3:])))
    return rows


def test_golden_values():
    rows = _golden_rows()
    assert len(rows) >= 20
    xin = np.array([r[0] for r in rows], dtype=np.uint32).view(np.float32)
    got = rn16(xin)
    for (xb, hb, val, src), g, w in zip(rows, got, widen(got)):
        assert int(g) == hb, f"rn16({xb:08x}) = {int(g):04x}, expected {hb:04x} ({src})"
        if math.isinf(val):
            assert math.isinf(float(w)) and math.copysign(1, float(w)) == math.copysign(1, val)
        else:
            assert float(w) == val and math.copysign(1, float(w)) == math.copysign(1, val), src


def _closed_form_half(h):
    s = -1.0 if h & 0x8000 else 1.0
    e = (h >> 10) & 0x1F
    m = h & 0x3FF
    if e == 0:
        return s * m * 2.0 ** -24
    if e == 31:
        return s * math.inf if m == 0 else math.nan
    return s * 2.0 ** (e - 15) * (1 + m / 1024)


def test_widen_exhaustive_closed_form():
    """All 65,536 binary16 patterns: widen == (-1)^s 2^(e-15)(1 + m/1024) (normal),
    (-1)^s m 2^-24 (subnormal); sign of zero kept; NaN stays NaN."""
    h = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    w = widen(h)
    for i in range(65536):
        ref = _closed_form_half(i)
        got = float(w[i])
        if math.isnan(ref):
            assert math.isnan(got), hex(i)
        else:
            assert got == ref and math.copysign(1, got) == math.copysign(1, ref), hex(i)


def test_widen_matches_struct_codec():
    """CPython's struct 'e' codec is an independent binary16 decoder."""
    h = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    w = widen(h)
    for i in range(0, 65536, 7):
        ref = struct.unpack("<e", struct.pack("<H", i))[0]
        if math.isnan(ref):
            assert math.isnan(float(w[i]))
        else:
            assert float(w[i]) == ref


def test_rn16_roundtrip_of_every_half():
    """rn16(widen(h)) == h for every non-NaN half (rounding an exactly
    representable value is the identity)."""
    h = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    e = (h.astype(np.int64) >> 10) & 0x1F
    m = h.astype(np.int64) & 0x3FF
    ok = ~((e == 31) & (m != 0))
    assert np.array_equal(rn16(widen(h))[ok], h[ok])


def _stratified_fp32_sample(seed=0, per_exp=24):
    """Every fp32 exponent, with random fractions plus the rounding-critical
    fractions: exact ties, one below and one above, all 13 dropped bits set."""
    g = np.random.default_rng([1605, 8325, 777, seed])
    bits = []
    for E in range(0, 256):
        fr = list(g.integers(0, 1 << 23, per_exp))
        for keep in (0, 1, 2, 0x3FF, 0x155):
            base = keep << 13
            fr += [base | 0x1000, base | 0x0FFF, base | 0x1001, base | 0x1FFF, base]
        for f in fr:
            for s in (0, 1):
                bits.append((s << 31) | (E << 23) | int(f))
    # subnormal-half ties at every shift: value = (2q+1) * 2^(shift-1) units
    for E in range(100, 113):
        shift = 126 - E
        for q in (0, 1, 2, 3, 511, 1022, 1023):
            sig = ((2 * q + 1) << (shift - 1)) if shift - 1 < 24 else None
            if sig is None or sig >= (1 << 24) or sig < (1 << 23):
                continue
            bits.append((E << 23) | (sig & 0x7FFFFF))
    return np.array(bits, dtype=np.uint32)


def test_rn16_vs_exact_rational_stratified():
    """rn16 against exact-rational round-half-even to binary16 (tests/exact.py)."""
    b = _stratified_fp32_sample()
    x = b.view(np.float32)
    finite = np.isfinite(x)
    x = x[finite]
    got = widen(rn16(x))
    for xi, gi in zip(x, got):
        ref = exact.to16(float(xi))
        gi = float(gi)
        assert gi == ref and math.copysign(1, gi) == math.copysign(1, ref), (float(xi), gi, ref)


def test_rn16_vs_struct_codec_random():
    """CPython's struct 'e' packer rounds half-to-even (PyFloat_Pack2); compare on
    random doubles that are fp32 values in the half range."""
    g = np.random.default_rng([1605, 8325, 778])
    x = np.concatenate([
        g.uniform(-65504, 65504, 20000),
        g.standard_normal(20000) * 1e-5,
        g.standard_normal(20000) * 1e-2,
    ]).astype(np.float32)
    got = rn16(x)
    for xi, gi in zip(x, got):
        ref = struct.unpack("<H", struct.pack("<e", float(xi)))[0]
        assert int(gi) == ref, (float(xi), hex(int(gi)), hex(ref))


def test_rn16_precision_bound():
    """|widen(rn16(x)) - x| <= 2^-11 max(|x|, 2^-14) in the finite range."""
    g = np.random.default_rng([1605, 8325, 779])
    x = np.concatenate([g.uniform(-65504, 65504, 100000), g.standard_normal(100000) * 1e-4]).astype(np.float32)
    err = np.abs(widen(rn16(x)).astype(np.float64) - x.astype(np.float64))
    bound = 2.0 ** -11 * np.maximum(np.abs(x.astype(np.float64)), 2.0 ** -14)
    assert np.all(err <= bound)


def test_overflow_threshold():
    x = np.array([65504, 65519.99, 65520, -65520, 1e30, np.inf, np.nan], dtype=np.float32)
    assert overflow16(x).tolist() == [False, False, True, True, True, False, False]
    h = rn16(x)
    assert (h[2] & 0x7FFF) == 0x7C00 and (h[3] & 0x7FFF) == 0x7C00
    assert (h[4] & 0x7FFF) == 0x7C00 and h[5] == 0x7C00
    assert (h[6] & 0x7C00) == 0x7C00 and (h[6] & 0x3FF) != 0


@pytest.mark.slow
def test_rn16_exhaustive_vs_numpy():
    """All 2^32 fp32 patterns (opt-in, TM_EXHAUSTIVE=1; minutes): rn16 equals
    numpy's float16 conversion on every finite input and on +-inf."""
    step = 1 << 24
    for start in range(0, 1 << 32, step):
        b = np.arange(start, start + step, dtype=np.uint64).astype(np.uint32)
        x = b.view(np.float32)
        ours = rn16(x)
        ref = x.astype(np.float16).view(np.uint16)
        fin = ~np.isnan(x)
        assert np.array_equal(ours[fin], ref[fin]), start
