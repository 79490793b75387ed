"""Pins for oracle/easgd.py (CPU only)."""

import numpy as np
import pytest

import exact
from oracle.easgd import easgd_sequence, easgd_update
from paper_1605_08325_b200.inputs import worker_buffer

F32 = np.float32


def test_spec_example():
    # alpha = 0.5, x = 2, centre 0 -> x' = 1, centre' = 1
    x, c = easgd_update(np.array([2.0], F32), np.array([0.0], F32), 0.5)
    assert x.tolist() == [1.0] and c.tolist() == [1.0]


def test_alpha_one_swaps():
    # alpha = 1: x' = c and c' = x whenever x - c is exact (integers here)
    g = np.random.default_rng(1)
    x = g.integers(-1000, 1000, 1000).astype(F32)
    c = g.integers(-1000, 1000, 1000).astype(F32)
    x2, c2 = easgd_update(x, c, 1.0)
    assert np.array_equal(x2, c) and np.array_equal(c2, x)


def test_alpha_half_meets_in_the_middle():
    # alpha = 0.5 on integers: both become the exact midpoint (one exchange)
    g = np.random.default_rng(2)
    x = g.integers(-1000, 1000, 1000).astype(F32)
    c = g.integers(-1000, 1000, 1000).astype(F32)
    x2, c2 = easgd_update(x, c, 0.5)
    mid = ((x.astype(np.float64) + c.astype(np.float64)) / 2).astype(F32)
    assert np.array_equal(x2, mid) and np.array_equal(c2, mid)


@pytest.mark.parametrize("alpha", [0.5, 0.0625, 0.3])
@pytest.mark.parametrize("dist", ["D1", "D2", "D3", "D6"])
def test_brute_force_steps(alpha, dist):
    """Each of d = x - c, e = alpha d, x' = x - e, c' = c + e is one correctly
    rounded fp32 operation (no FMA), checked with exact rationals."""
    x = worker_buffer(64, dist, 0, config=21)
    c = worker_buffer(64, dist, 1, config=21)
    x2, c2 = easgd_update(x, c, alpha)
    a = float(F32(alpha))
    for i in range(64):
        d = exact.sub(x[i], c[i])
        e = exact.mul(a, d)
        assert exact.same_bits32(x2[i], exact.sub(x[i], e)), (i, x[i], c[i])
        assert exact.same_bits32(c2[i], exact.add(c[i], e))


@pytest.mark.parametrize("alpha", [0.5, 0.0625, 0.3])
def test_conservation(alpha):
    """x + c is conserved exactly in rational arithmetic ((x-e)+(c+e) = x+c) and
    within one rounding of each output in fp32: |(x'+c')-(x+c)| <= 2^-24(|x'|+|c'|)."""
    x = worker_buffer(200000, "D1", 0, config=22)
    c = worker_buffer(200000, "D1", 1, config=22)
    x2, c2 = easgd_update(x, c, alpha)
    lhs = np.abs((x2.astype(np.float64) + c2) - (x.astype(np.float64) + c))
    assert np.all(lhs <= 2.0 ** -24 * (np.abs(x2.astype(np.float64)) + np.abs(c2)))


def test_sequence_is_ordered_composition():
    """'Without the Round-Robin scheme': updates apply one at a time
    in arrival order; the sequence equals the explicit composition, and a
    different order gives a different (valid) centre."""
    ws = [worker_buffer(1000, "D1", r, config=23) for r in range(4)]
    c = worker_buffer(1000, "D1", 9, config=23)
    order = [2, 0, 3, 1, 2]
    nws, nc = easgd_sequence(ws, c, 0.125, order)
    ref = [w.copy() for w in ws]
    cc = c.copy()
    for w in order:
        ref[w], cc = easgd_update(ref[w], cc, 0.125)
    assert np.array_equal(nc, cc)
    for a, b in zip(nws, ref):
        assert np.array_equal(a, b)
    _, nc2 = easgd_sequence(ws, c, 0.125, [0, 1, 2, 3, 2])
    assert not np.array_equal(nc, nc2)
    # conservation across a whole round: sum_w x_w + c conserved up to rounding
    tot0 = sum(w.astype(np.float64) for w in ws) + c
    tot1 = sum(w.astype(np.float64) for w in nws) + nc
    assert np.max(np.abs(tot1 - tot0)) < 1e-5


def test_quadratic_steps_brute_force():
    """Each local step of the synthetic objective is d = fl(x - t),
    x = fl(x - fl(eta d)): exact-rational emulation over 3 steps."""
    from oracle.easgd import quadratic_sgd_steps
    x = worker_buffer(48, "D1", 0, config=24)
    t = worker_buffer(48, "D1", 1, config=24)
    for eta in (0.25, 0.3):
        got = quadratic_sgd_steps(x, t, eta, 3)
        e = float(F32(eta))
        for i in range(48):
            xi = float(x[i])
            for _ in range(3):
                xi = exact.sub(xi, exact.mul(e, exact.sub(xi, float(t[i]))))
            assert exact.same_bits32(got[i], xi), (eta, i)


def test_quadratic_steps_closed_form():
    """eta = 1/2 on dyadic inputs is exact: x_tau - t = (x_0 - t) / 2^tau."""
    from oracle.easgd import quadratic_sgd_steps
    g = np.random.default_rng(25)
    x = (g.integers(-2 ** 12, 2 ** 12, 500) * 2.0 ** -4).astype(F32)
    t = (g.integers(-2 ** 12, 2 ** 12, 500) * 2.0 ** -4).astype(F32)
    got = quadratic_sgd_steps(x, t, 0.5, 4)
    want = t.astype(np.float64) + (x.astype(np.float64) - t) / 16.0
    assert np.array_equal(got.astype(np.float64), want)


def test_async_replay_reduces_and_converges():
    """tau = 0 is the plain arrival-order sequence; with local steps the loop is
    the explicit composition; and with all targets equal to t and many rounds the
    centre and every worker converge to t (EASGD's fixed point)."""
    from oracle.easgd import easgd_async_replay, quadratic_sgd_steps
    ws = [worker_buffer(500, "D1", r, config=26) for r in range(3)]
    ts = [worker_buffer(500, "D1", 10 + r, config=26) for r in range(3)]
    c = worker_buffer(500, "D1", 9, config=26)
    order = [1, 0, 2, 1, 2, 0]
    a_w, a_c = easgd_async_replay(ws, c, ts, 0.25, 0, 0.125, order)
    b_w, b_c = easgd_sequence(ws, c, 0.125, order)
    assert np.array_equal(a_c, b_c) and all(np.array_equal(p, q) for p, q in zip(a_w, b_w))
    a_w, a_c = easgd_async_replay(ws, c, ts, 0.25, 2, 0.125, order)
    ref = [w.copy() for w in ws]
    cc = c.copy()
    for w in order:
        ref[w] = quadratic_sgd_steps(ref[w], ts[w], 0.25, 2)
        ref[w], cc = easgd_update(ref[w], cc, 0.125)
    assert np.array_equal(a_c, cc) and all(np.array_equal(p, q) for p, q in zip(a_w, ref))
    t = worker_buffer(500, "D1", 20, config=26)
    f_w, f_c = easgd_async_replay(ws, c, [t] * 3, 0.5, 1, 0.5, [0, 1, 2] * 60)
    assert np.max(np.abs(f_c.astype(np.float64) - t)) < 1e-6
    assert all(np.max(np.abs(w.astype(np.float64) - t)) < 1e-6 for w in f_w)


from hypothesis import given, settings, strategies as st  # noqa: E402

_F32_1E37 = float(np.float32(1e37))


@settings(max_examples=300, deadline=None)
@given(x=st.lists(st.floats(width=32, min_value=-_F32_1E37, max_value=_F32_1E37), min_size=1, max_size=6),
       c=st.floats(width=32, min_value=-_F32_1E37, max_value=_F32_1E37),
       alpha=st.sampled_from([0.5, 0.0625, 0.3, 1.0, 0.125]))
def test_property_update_vs_brute_force(x, c, alpha):
    """Any finite fp32 worker / centre values (subnormals, mixed magnitudes):
    each of the four steps is one correctly rounded operation."""
    xs = np.array(x, dtype=F32)
    cs = np.full(len(x), c, dtype=F32)
    x2, c2 = easgd_update(xs, cs, alpha)
    a = float(F32(alpha))
    for i in range(len(x)):
        d = exact.sub(float(xs[i]), float(cs[i]))
        e = exact.mul(a, d)
        assert exact.same_bits32(x2[i], exact.sub(float(xs[i]), e))
        assert exact.same_bits32(c2[i], exact.add(float(cs[i]), e))


# ---------------------------------------------------------------------------
# Concurrent updates: easgd_interleavings / easgd_concurrent_admissible (Q15)
# ---------------------------------------------------------------------------
import itertools as _it  # noqa: E402
import math as _math  # noqa: E402
import os as _os  # noqa: E402

from oracle.easgd import easgd_concurrent_admissible, easgd_interleavings  # noqa: E402


def _golden_interleavings():
    path = _os.path.join(_os.path.dirname(__file__), "golden", "easgd_interleavings.txt")
    cases, cur = [], None
    for line in open(path):
        line = line.split("#")[0].strip()
        if not line:
            continue
        if line.startswith("case"):
            cur = ([float(v) for v in line.split()[1:]], set())
            cases.append(cur)
        else:
            cur[1].add(tuple(float(v) for v in line.split()))
    return cases


def test_interleavings_golden_two_workers():
    """The distinct results equal the hand-derived sets (tests/golden/
    easgd_interleavings.txt, SPEC L475 + PAPER L573-581)."""
    cases = _golden_interleavings()
    assert len(cases) == 2
    for (xa, xb, c, alpha), want in cases:
        got = {(float(ws[0][0]), float(ws[1][0]), float(cc[0]))
               for ws, cc in easgd_interleavings([np.float32([xa]), np.float32([xb])], np.float32([c]), alpha)}
        assert got == want


@pytest.mark.parametrize("n", [1, 2, 3, 4])
def test_interleavings_path_count(n):
    X = [worker_buffer(5, "D1", r, config=70) for r in range(n)]
    c = worker_buffer(5, "D1", 9, config=70)
    assert len(easgd_interleavings(X, c, 0.3)) == _math.factorial(n) ** 2


def test_interleavings_one_worker_is_the_update():
    x, c = worker_buffer(1000, "D2", 0, config=71), worker_buffer(1000, "D2", 1, config=71)
    (ws, cc), = easgd_interleavings([x], c, 0.3)
    wx, wc = easgd_update(x, c, 0.3)
    assert np.array_equal(ws[0].view(np.uint32), wx.view(np.uint32))
    assert np.array_equal(cc.view(np.uint32), wc.view(np.uint32))


@pytest.mark.parametrize("n", [2, 3, 4])
def test_every_arrival_order_is_admissible(n):
    """A serial arrival order (each worker reads the centre after all earlier adds)
    is one of the interleavings: easgd_sequence's result is a member everywhere."""
    P = 4000
    X = [worker_buffer(P, "D1", r, config=72) for r in range(n)]
    c = worker_buffer(P, "D1", 9, config=72)
    for order in _it.permutations(range(n)):
        ws, cc = easgd_sequence(X, c, 0.3, list(order))
        assert easgd_concurrent_admissible(X, c, 0.3, ws, cc).all()


def test_stale_reads_are_admissible_but_lost_or_doubled_updates_are_not():
    """All workers reading the initial centre (every update stale) is admissible;
    dropping one worker's add, adding one twice, or an FMA-contracted update is
    not (on generic inputs: fails on most elements)."""
    P, n, a = 4000, 3, np.float32(0.3)
    X = [worker_buffer(P, "D1", r, config=73) for r in range(n)]
    c = worker_buffer(P, "D1", 9, config=73)
    es = [np.multiply(a, np.subtract(x, c, dtype=np.float32), dtype=np.float32) for x in X]
    stale_w = [np.subtract(x, e, dtype=np.float32) for x, e in zip(X, es)]
    cc = c
    for e in es:
        cc = np.add(cc, e, dtype=np.float32)
    assert easgd_concurrent_admissible(X, c, a, stale_w, cc).all()
    lost = np.add(np.add(c, es[0], dtype=np.float32), es[1], dtype=np.float32)
    assert easgd_concurrent_admissible(X, c, a, stale_w, lost).mean() < 0.05
    doubled = np.add(cc, es[2], dtype=np.float32)
    assert easgd_concurrent_admissible(X, c, a, stale_w, doubled).mean() < 0.05
    # FMA contraction of x' = x - alpha (x - c): one rounding instead of two
    fma_w = [np.float32(np.float64(x) - np.float64(a) * np.float64(np.subtract(x, c, dtype=np.float32)))
             for x in X]
    fma_w = [np.asarray(w, dtype=np.float32) for w in fma_w]
    assert easgd_concurrent_admissible(X, c, a, fma_w, cc).mean() < 0.9


def test_ftz_add_flushes_subnormals():
    """The `ftz` centre add (model of the hardware float atomic, Q15) flushes a
    subnormal sum to signed zero; the IEEE add keeps it."""
    tiny = np.float32(2.0 ** -130)
    x, c = np.float32([2 * tiny]), np.float32([0.0])  # e = alpha * 2 tiny = tiny (alpha = 1/2)
    ieee = {float(cc[0]) for _, cc in easgd_interleavings([x], c, 0.5, add="ieee")}
    ftz = {float(cc[0]) for _, cc in easgd_interleavings([x], c, 0.5, add="ftz")}
    assert ieee == {float(tiny)} and ftz == {0.0}
