"""Pins for oracle/bsp.py (CPU only)."""

import numpy as np
import pytest

import exact
from oracle import exchange as ox
from oracle.bsp import bsp_iteration, sgd_step
from paper_1605_08325_b200.inputs import worker_buffer, worker_buffers

F32 = np.float32


def test_spec_examples():
    # mu = 0, lr = 0.1, w = [0], g = [1] -> w = [-0.1]
    w, v = sgd_step(np.array([0.0], F32), np.array([0.0], F32), np.array([1.0], F32), 0.1, 0.0)
    assert w[0] == F32(-0.1) and v[0] == F32(-0.1)
    # g = 0 (and v = 0) -> weights unchanged, velocity decayed by mu
    x = worker_buffer(1000, "D1", 0, config=30)
    v0 = worker_buffer(1000, "D1", 1, config=30)
    w, v = sgd_step(x, np.zeros_like(x), np.zeros_like(x), 0.1, 0.9)
    assert np.array_equal(w, x)
    w, v = sgd_step(x, v0, np.zeros_like(x), 0.1, 0.9)
    assert np.array_equal(v, (F32(0.9) * v0).astype(F32))


def test_three_steps_match_exact_unrolled_recurrence():
    """3 steps with mu = 0.9 against a hand-unrolled recurrence in
    exact rationals with one fp32 rounding per operation."""
    g = worker_buffers(16, 3, "D2", config=31)
    w = worker_buffer(16, "D1", 5, config=31)
    v = np.zeros(16, F32)
    lr, mu = 0.05, 0.9
    W, Vv = w.copy(), v.copy()
    for t in range(3):
        W, Vv = sgd_step(W, Vv, g[t], lr, mu)
    for i in range(16):
        wi, vi = float(w[i]), 0.0
        for t in range(3):
            vi = exact.sub(exact.mul(float(F32(mu)), vi), exact.mul(float(F32(lr)), g[t][i]))
            wi = exact.add(wi, vi)
        assert exact.same_bits32(W[i], wi) and exact.same_bits32(Vv[i], vi)


@pytest.mark.parametrize("strategy", ["asa", "asa16", "ar"])
def test_bsp_iteration_composes_step_and_exchange(strategy):
    k, P = 4, 1001
    W = worker_buffers(P, k, "D2", config=32)
    V = worker_buffers(P, k, "D4", config=33)
    G = worker_buffers(P, k, "D2", config=34)
    W2, V2 = bsp_iteration(W, V, G, 0.01, 0.9, strategy, exchange_momentum=True)
    W1 = [sgd_step(W[j], V[j], G[j], 0.01, 0.9)[0] for j in range(k)]
    V1 = [sgd_step(W[j], V[j], G[j], 0.01, 0.9)[1] for j in range(k)]
    want_w, want_v = ox.exchange(W1, strategy), ox.exchange(V1, strategy)
    for j in range(k):
        assert np.array_equal(W2[j], want_w[j]) and np.array_equal(V2[j], want_v[j])
    _, V3 = bsp_iteration(W, V, G, 0.01, 0.9, strategy, exchange_momentum=False)
    for j in range(k):
        assert np.array_equal(V3[j], V1[j])
    # lockstep: after the exchange all workers hold identical weights
    for j in range(1, k):
        assert np.array_equal(W2[j], W2[0])
