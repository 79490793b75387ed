"""Pins for oracle/exchange.py (CPU only).

Each test checks the oracle against something other than itself: SPEC worked
examples, exact-rational emulation of every rounding step (tests/exact.py),
closed forms in exact arithmetic, and proven error bounds (Q11, Q12).
"""

import math
from fractions import Fraction

import numpy as np
import pytest

import exact
from oracle import exchange as ex
from oracle.fp16 import rn16, widen
from paper_1605_08325_b200.inputs import DISTS, dyadic_buffers, worker_buffers

F32 = np.float32


def bits(a):
    return np.asarray(a, dtype=np.float32).view(np.uint32)


def assert_bitwise(a, b, msg=""):
    a, b = np.asarray(a, np.float32), np.asarray(b, np.float32)
    assert a.shape == b.shape
    ok = (bits(a) == bits(b)) | (np.isnan(a) & np.isnan(b))
    assert ok.all(), f"{msg}: {np.count_nonzero(~ok)} mismatches, first at {np.argmax(~ok)}"


# --------------------------------------------------------------------- layout

@pytest.mark.parametrize("k", range(1, 17))
def test_partition_roundtrip_and_padding(k):
    g = np.random.default_rng([1605, k])
    for P in (1, 2, 5, 7, 100, 1023, 10000):
        x = g.standard_normal(P).astype(F32)
        sl = ex.partition(x, k)
        L = -(-P // k)
        assert len(sl) == k and all(s.shape == (L,) for s in sl)
        assert_bitwise(ex.unpartition(sl, P), x)
        pad = np.concatenate(sl)[P:]
        assert np.all(bits(pad) == 0)  # +0 padding


def test_partition_spec_examples():
    # SPEC L81-82
    a = np.arange(1, 5, dtype=F32)
    s = ex.partition(a, 2)
    assert s[0].tolist() == [1, 2] and s[1].tolist() == [3, 4]
    s = ex.partition(np.arange(1, 6, dtype=F32), 2)
    assert s[0].tolist() == [1, 2, 3] and s[1].tolist() == [4, 5, 0]


def test_alltoall_transpose():
    # 2-rank transpose; transpose o transpose == identity
    send = [["A0", "A1"], ["B0", "B1"]]
    assert ex.alltoall(send) == [["A0", "B0"], ["A1", "B1"]]
    for k in (1, 3, 8):
        send = [[(j, r) for r in range(k)] for j in range(k)]
        assert ex.alltoall(ex.alltoall(send)) == send


# --------------------------------------------------------------- worked values

def test_spec_asa_example_k2():
    # sums [11,22,33,44]; averaged (AWAGD) -> [5.5,11,16.5,22]
    X = [np.array([1, 2, 3, 4], F32), np.array([10, 20, 30, 40], F32)]
    for strat in ("ar", "asa", "asa16"):
        out = ex.exchange(X, strat)
        for o in out:
            assert o.tolist() == [5.5, 11.0, 16.5, 22.0], strat


def test_spec_awagd_example():
    # [0.2], [0.6] -> [0.4] (fp32: fl(fl(0.2+0.6)/2) == 0.4f)
    X = [np.array([0.2], F32), np.array([0.6], F32)]
    for o in ex.asa_average(X):
        assert bits(o)[0] == bits(np.array([0.4], F32))[0]


def test_spec_asa16_example():
    # k=2, [0.1]+[0.1] -> sum 0.199951171875, average 0.0999755859375
    X = [np.array([0.1], F32), np.array([0.1], F32)]
    for o in ex.asa16_average(X):
        assert float(o[0]) == 0.0999755859375


def test_spec_k3_integers_padding_path():
    # k = 3, P = 7, integer-valued floats: the sum is exact, so the
    # average is the correctly rounded exact mean.
    g = np.random.default_rng([1605, 3])
    X = [g.integers(-1000, 1000, 7).astype(F32) for _ in range(3)]
    exact_sum = [sum(int(x[i]) for x in X) for i in range(7)]
    want = np.array([exact.div(s, 3) for s in exact_sum], F32)
    for strat in ("ar", "asa"):
        for o in ex.exchange(X, strat):
            assert_bitwise(o, want, strat)


def test_k1_identity():
    # SPEC L488/L555, reading Q10: k = 1 returns the input for every strategy
    x = worker_buffers(1000, 1, "D6")[0]
    for strat in ex.STRATEGIES:
        assert_bitwise(ex.exchange([x], strat)[0], x, strat)


# ------------------------------------------------- exact-rational brute force

def _brute_asa(values, k):
    s = float(values[0])
    for j in range(1, k):
        s = exact.add(s, values[j])
    return exact.div(s, k)


def _brute_asa16(values, k):
    h = [exact.to16(v) for v in values]
    s = h[0]
    for j in range(1, k):
        s = exact.add(s, h[j])
    a = exact.div(s, k)
    return exact.to16(a)


@pytest.mark.parametrize("dist", DISTS)
@pytest.mark.parametrize("k", [2, 3, 4, 5, 8])
def test_brute_force_every_rounding_step(dist, k):
    """P <= 8, k <= 8: each element recomputed with exact rationals and one
    correct rounding per step, in the paper's order (Fig. 2: sum over the k
    sub-arrays on the owner, then 1/k; Sec. 3.2 fp16 transfer)."""
    for P in (1, 5, 8):
        X = worker_buffers(P, k, dist, config=11)
        o_asa = ex.asa_average(X)
        o_ar = ex.ar_average(X)
        o_16 = ex.asa16_average(X)
        for i in range(P):
            vals = [float(x[i]) for x in X]
            want = _brute_asa(vals, k)
            want16 = _brute_asa16(vals, k)
            for r in range(k):
                assert exact.same_bits32(o_asa[r][i], want), (dist, k, P, i, vals)
                assert exact.same_bits32(o_ar[r][i], want)
                assert exact.same_bits32(o_16[r][i], want16), (dist, k, P, i, vals)


def test_signed_zero_rules():
    """Reading Q5: the sum starts at the rank-0 term, so all -0 inputs give -0;
    mixed +-0 give +0 (IEEE RN)."""
    nz = np.array([-0.0], F32)
    pz = np.array([0.0], F32)
    for strat in ("asa", "asa16"):
        assert bits(ex.exchange([nz, nz, nz, nz], strat)[0])[0] == 0x80000000
        assert bits(ex.exchange([nz, pz], strat)[0])[0] == 0


# --------------------------------------------------- closed forms / invariants

@pytest.mark.parametrize("k", [2, 4, 8])
def test_ar_equals_asa_equals_exact_mean_on_dyadics(k):
    """North star invariant 'AR equals ASA in exact arithmetic': with dyadic
    inputs m * 2^-10, |m| <= 512, every partial sum is exact for k <= 8, and the
    division by k = 2^n is exact, so both equal the exact mean bitwise."""
    X = dyadic_buffers(4099, k)
    exact_mean = (np.sum(np.stack(X).astype(np.float64), axis=0) / k).astype(F32)
    for strat in ("ar", "asa"):
        for o in ex.exchange(X, strat):
            assert_bitwise(o, exact_mean, strat)


@pytest.mark.parametrize("k", [2, 4, 8])
def test_asa16_equals_asa_on_small_integers(k):
    """Integers in [-256, 256]: fp16-exact inputs, |sum| <= 2048, averages are
    multiples of 1/8 with <= 11 significant bits -> ASA16 == ASA == exact mean."""
    X = worker_buffers(10007, k, "D5")
    exact_mean = (np.sum(np.stack(X).astype(np.float64), axis=0) / k).astype(F32)
    for o16, o in zip(ex.asa16_average(X), ex.asa_average(X)):
        assert_bitwise(o16, exact_mean)
        assert_bitwise(o, exact_mean)


def test_identity_of_identical_buffers():
    """fp32: k identical buffers give x back bitwise for k in {1,2,4}; for k = 8
    when x has <= 21 significant bits (j*x exact for j <= 8).  ASA16: identical
    buffers give widen(rn16(x)) for every k <= 8 (SURVEY finding 5)."""
    x = worker_buffers(20000, 1, "D1")[0]
    for k in (1, 2, 4):
        for o in ex.asa_average([x] * k):
            assert_bitwise(o, x)
    x21 = (x.view(np.uint32) & np.uint32(0xFFFFFFF8)).view(F32)
    for o in ex.asa_average([x21] * 8):
        assert_bitwise(o, x21)
    for k in range(2, 9):
        for o in ex.asa16_average([x] * k):
            assert_bitwise(o, widen(rn16(x)))


def test_cross_rank_identity():
    """every rank returns bitwise-identical buffers."""
    X = worker_buffers(3001, 8, "D2")
    for strat in ex.STRATEGIES:
        out = ex.exchange(X, strat)
        for o in out[1:]:
            assert_bitwise(o, out[0])


def test_segmentation_independence():
    """Reading Q7: the result is elementwise; it does not depend on the
    sub-array length (pad to ceil(P/k) or any larger L)."""
    X = worker_buffers(1000, 4, "D1")
    ref = ex.asa16_average(X)[0]
    el = ex.element_average(np.stack(X), "asa16")
    assert_bitwise(ref, el)
    ref = ex.asa_average(X)[0]
    assert_bitwise(ref, ex.element_average(np.stack(X), "asa"))


# --------------------------------------------------------------- error bounds

def _m(X):
    return np.mean(np.abs(np.stack(X).astype(np.float64)), axis=0)


@pytest.mark.parametrize("dist", ["D1", "D2", "D3", "D4"])
@pytest.mark.parametrize("k", [2, 4, 8])
def test_q11_order_bound(dist, k):
    """Reading Q11 (the tolerance for a GPU AR whose summation order is not
    fixed): any other order differs from the rank-order result by at most
    2(k-1) 2^-24 m_i <= 1e-6 m_i, m_i = mean_j |x_ij|.  Checked with the reverse
    and a shuffled order."""
    X = worker_buffers(50000, k, dist, config=5)
    ref = ex.ar_average(X)[0].astype(np.float64)
    m = _m(X)
    for order in (list(range(k))[::-1], list(np.random.default_rng(k).permutation(k))):
        other = ex.ar_average([X[j] for j in order])[0].astype(np.float64)
        assert np.all(np.abs(other - ref) <= 1e-6 * m)


@pytest.mark.parametrize("dist", ["D1", "D2", "D3", "D4"])
@pytest.mark.parametrize("k", [2, 4, 8])
def test_q12_asa16_bound(dist, k):
    """Reading Q12: |asa16_i - exact mean_i| <= 2^-10 m_i (1 + 2^-9) + 2^-24."""
    X = worker_buffers(50000, k, dist, config=6)
    out = ex.asa16_average(X)[0].astype(np.float64)
    mean = np.mean(np.stack(X).astype(np.float64), axis=0)
    m = _m(X)
    assert np.all(np.abs(out - mean) <= 2.0 ** -10 * m * (1 + 2.0 ** -9) + 2.0 ** -24)


def test_asa_vs_exact_mean_bound():
    """fp32 ASA is within (k-1) 2^-24 m + 2^-24 |mean| of the exact mean."""
    k = 8
    X = worker_buffers(50000, k, "D1", config=7)
    out = ex.asa_average(X)[0].astype(np.float64)
    mean = np.mean(np.stack(X).astype(np.float64), axis=0)
    m = _m(X)
    assert np.all(np.abs(out - mean) <= (k - 1) * 2.0 ** -24 * m + 2.0 ** -24 * np.abs(mean) + 1e-45)


# ------------------------------------------------------------ traffic counting

def test_traffic_accounting_spec():
    # P = 1024, k = 4 -> ASA 6144 B, ASA16 3072 B per rank
    assert ex.wire_bytes_per_rank("asa", 1024, 4) == 6144
    assert ex.wire_bytes_per_rank("asa16", 1024, 4) == 3072
    for P in (1, 7, 1000003):
        for k in (2, 4, 8):
            assert 2 * ex.wire_bytes_per_rank("asa16", P, k) == ex.wire_bytes_per_rank("asa", P, k)
            assert ex.wire_bytes_per_rank("asa", P, k) == 2 * (k - 1) * (-(-P // k)) * 4
    assert ex.wire_bytes_per_rank("asa16", 123, 1) == 0


# ------------------------------------------------------------- SUBGD sum mode

def test_spec_sum_examples():
    # k=2 [1,2,3,4] + [10,20,30,40] -> sums [11,22,33,44]
    X = [np.array([1, 2, 3, 4], F32), np.array([10, 20, 30, 40], F32)]
    for strat in ("ar", "asa", "asa16"):
        for o in ex.exchange(X, strat, op="sum"):
            assert o.tolist() == [11.0, 22.0, 33.0, 44.0], strat
    # k=2, [0.1] + [0.1] in ASA16 -> 0.199951171875
    X = [np.array([0.1], F32), np.array([0.1], F32)]
    for o in ex.asa16_average(X, op="sum"):
        assert float(o[0]) == 0.199951171875


def _brute_sum(values, k, q16):
    h = [exact.to16(v) if q16 else float(v) for v in values]
    s = h[0]
    for j in range(1, k):
        s = exact.add(s, h[j])
    return exact.to16(s) if q16 else s


@pytest.mark.parametrize("dist", DISTS)
@pytest.mark.parametrize("k", [2, 3, 5, 8])
def test_sum_brute_force(dist, k):
    for P in (1, 6):
        X = worker_buffers(P, k, dist, config=12)
        o = ex.asa_average(X, op="sum")
        o16 = ex.asa16_average(X, op="sum")
        oar = ex.ar_average(X, op="sum")
        for i in range(P):
            vals = [float(x[i]) for x in X]
            assert exact.same_bits32(o[1][i], _brute_sum(vals, k, False))
            assert exact.same_bits32(oar[0][i], _brute_sum(vals, k, False))
            assert exact.same_bits32(o16[k - 1][i], _brute_sum(vals, k, True))


@pytest.mark.parametrize("k", [2, 4, 8])
def test_sum_is_k_times_average_for_power_of_two_k(k):
    """For k = 2^n, fl(s / k) = s / k exactly for normal s, so the SUBGD sum is
    k times the AWAGD average bitwise (D1: no fp32 subnormal averages)."""
    X = worker_buffers(20000, k, "D1", config=13)
    s = ex.asa_average(X, op="sum")[0]
    a = ex.asa_average(X)[0]
    assert_bitwise(s, (a.astype(np.float64) * k).astype(F32))


@pytest.mark.parametrize("k", [2, 4, 8])
def test_asa16_sum_exact_on_small_integers(k):
    """Integers in [-256, 256]: every partial sum is an integer of magnitude <=
    2048, exact in binary16, so the ASA16 sum is the exact sum."""
    X = worker_buffers(5001, k, "D5", config=14)
    exact_sum = np.sum(np.stack(X).astype(np.float64), axis=0).astype(F32)
    for o in ex.asa16_average(X, op="sum"):
        assert_bitwise(o, exact_sum)


# Property-based pin (hypothesis): fp32 values drawn over the whole finite range
# the arithmetic stays finite in -- fp32 subnormals, binary16 subnormals and
# ties, values up to the binary16 limit (ASA16) or 1e37 (ASA), mixed magnitudes
# and signs -- against the exact-rational brute force of the same steps.
from hypothesis import given, settings, strategies as st  # noqa: E402

_F32_1E37 = float(np.float32(1e37))
_F16_LIM = float(np.float32(65519.99))  # largest fp32 below the binary16 overflow threshold 65520
_f32_asa = st.floats(width=32, min_value=-_F32_1E37, max_value=_F32_1E37)
_f32_asa16 = st.floats(width=32, min_value=-_F16_LIM, max_value=_F16_LIM)


def _cols(elem):
    return st.lists(st.lists(elem, min_size=8, max_size=8), min_size=1, max_size=3)


@settings(max_examples=300, deadline=None)
@given(k=st.integers(2, 8), cols=_cols(_f32_asa))
def test_property_asa_vs_brute_force(k, cols):
    X = [np.array([c[j] for c in cols], dtype=F32) for j in range(k)]
    o = ex.asa_average(X)
    for i in range(len(cols)):
        vals = [float(x[i]) for x in X]
        assert exact.same_bits32(o[0][i], _brute_asa(vals, k)), (k, vals)


@settings(max_examples=300, deadline=None)
@given(k=st.integers(2, 8), cols=_cols(_f32_asa16))
def test_property_asa16_vs_brute_force(k, cols):
    X = [np.array([c[j] for c in cols], dtype=F32) for j in range(k)]
    o = ex.asa16_average(X)
    for i in range(len(cols)):
        vals = [float(x[i]) for x in X]
        assert exact.same_bits32(o[0][i], _brute_asa16(vals, k)), (k, vals)
