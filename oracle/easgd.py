"""Elastic-averaging SGD (EASGD) worker/centre update.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Paper anchors: PAPER.md L143-148 (Sec. 2: "an elastic averaging strategy between
asynchronous workers and the server") and L573-588 (Sec. 4: EASGD re-implemented on
CUDA-aware MPI SendRecv() "without the Round-Robin scheme"; alpha = 0.5, tau = 1).
The paper does not print the update (reading Q13); SPEC.md L475 gives the
symmetric elastic update with one shared elastic difference:

    e  = alpha * (x_i - c)        x_i <- x_i - e        c <- c + e

Here each line is one fp32 operation with no FMA (reading Q13):
    d = fl(x - c);  e = fl(alpha * d);  x' = fl(x - e);  c' = fl(c + e).

"Without the Round-Robin scheme" (reading Q15): the server applies workers'
updates one at a time in ARRIVAL order; easgd_sequence takes that order
explicitly.

The asynchronous loop around the update:
each worker takes tau local SGD steps, then exchanges elastically with the centre;
the centre serves the exchanges one at a time in arrival order.  The model's
gradient is outside this repo's scope; easgd_async_replay uses the synthetic
quadratic objective f_w(x) = |x - t_w|^2 / 2 (gradient x - t_w), one fp32 rounding
per operation: d = fl(x - t); x = fl(x - fl(eta * d)).

Parity status: easgd_update and easgd_sequence are pinned
(tests/test_oracle_easgd.py: SPEC L478 example, alpha = 1 swap-converge, exact
rational brute force of each rounding step, conservation of x + c in exact
arithmetic and within one rounding in fp32).

Concurrent updates (reading Q15: several workers update one centre at once,
each reading a possibly stale c, the adds atomic -- "without the Round-Robin
scheme", L573-581) have no single result.  easgd_interleavings enumerates
every result they can produce -- every order of the atomic adds and every
state of c each worker can have read -- and easgd_concurrent_admissible tests
a result for membership, element by element.  Pinned (tests/test_oracle_easgd.py)
by the hand-derived two-worker example of tests/golden/easgd_interleavings.txt,
by N = 1 reducing to easgd_update, by every arrival order of easgd_sequence
being a member, by the path count N!^2, and by lost updates, a second add of one
worker and an FMA-contracted update failing membership.  The `ftz` add models
the hardware float atomic of the fast concurrent mode (PTX red.add.f32 flushes
subnormal operands and results to sign-preserving zero; reading Q15).
"""

import itertools

import numpy as np


def easgd_update(x, c, alpha):
    """One elastic update.  x, c: float32 arrays (same shape); alpha: float.
    Returns (x', c')."""
    x = np.asarray(x, dtype=np.float32)
    c = np.asarray(c, dtype=np.float32)
    a = np.float32(alpha)
    d = np.subtract(x, c, dtype=np.float32)
    e = np.multiply(a, d, dtype=np.float32)
    x_new = np.subtract(x, e, dtype=np.float32)
    c_new = np.add(c, e, dtype=np.float32)
    return x_new, c_new


def easgd_sequence(workers, center, alpha, order):
    """Apply the elastic update of workers[w] for w in `order` (arrival order),
    one after the other, against the shared centre.  Returns (new_workers,
    new_center); inputs are not modified."""
    ws = [np.array(w, dtype=np.float32, copy=True) for w in workers]
    c = np.array(center, dtype=np.float32, copy=True)
    for w in order:
        ws[w], c = easgd_update(ws[w], c, alpha)
    return ws, c


def quadratic_sgd_steps(x, t, eta, tau):
    """tau SGD steps on |x - t|^2 / 2, one fp32 rounding per operation."""
    x = np.array(x, dtype=np.float32, copy=True)
    t = np.asarray(t, dtype=np.float32)
    e = np.float32(eta)
    for _ in range(tau):
        d = np.subtract(x, t, dtype=np.float32)
        x = np.subtract(x, np.multiply(e, d, dtype=np.float32), dtype=np.float32)
    return x


def easgd_async_replay(workers, center, targets, eta, tau, alpha, order):
    """The asynchronous EASGD loop replayed in a given arrival order: for each
    worker id w in `order`, worker w first takes tau local steps from where its
    previous exchange left it, then applies the elastic update against the
    current centre.  Returns (new_workers, new_center)."""
    ws = [np.array(w, dtype=np.float32, copy=True) for w in workers]
    c = np.array(center, dtype=np.float32, copy=True)
    for w in order:
        ws[w] = quadratic_sgd_steps(ws[w], targets[w], eta, tau)
        ws[w], c = easgd_update(ws[w], c, alpha)
    return ws, c


def _ftz(v):
    """Sign-preserving flush of fp32 subnormals to zero."""
    v = np.asarray(v, dtype=np.float32)
    return np.where(np.abs(v) < np.float32(2.0 ** -126), np.copysign(np.float32(0.0), v), v).astype(np.float32)


def _centre_add(c, e, add):
    """One atomic centre add: "ieee" = fl(c + e); "ftz" = the hardware float
    atomic (subnormal operands and result flushed, reading Q15)."""
    if add == "ieee":
        return np.add(c, e, dtype=np.float32)
    if add == "ftz":
        return _ftz(np.add(_ftz(c), _ftz(e), dtype=np.float32))
    raise ValueError(add)


def easgd_interleavings(workers, center, alpha, add="ieee"):
    """Every result N CONCURRENT elastic updates of one centre can produce
    (reading Q15), as a list of (new_workers, new_center), one per path.

    A path is an order sigma of the N atomic centre adds plus, for the worker
    whose add comes t-th, the state of c it read: c_r with 0 <= r <= t (c_0 the
    initial centre, c_{t+1} = add(c_t, e_sigma(t))) -- a worker reads before its
    own add, and an atomic centre only ever holds one of the c_t.  Worker w then
    computes, as in easgd_update, d = fl(x_w - c_r), e_w = fl(alpha d),
    x_w' = fl(x_w - e_w).  N! orders times t+1 read choices per position: N!^2
    paths (1, 4, 36, 576 for N = 1..4)."""
    ws0 = [np.asarray(w, dtype=np.float32) for w in workers]
    c0 = np.asarray(center, dtype=np.float32)
    a = np.float32(alpha)
    n = len(ws0)
    if not 1 <= n <= 4:
        raise ValueError("interleavings are enumerated for 1..4 workers")
    out = []
    for sigma in itertools.permutations(range(n)):
        for reads in itertools.product(*[range(t + 1) for t in range(n)]):
            states = [c0]
            ws = list(ws0)
            for t, w in enumerate(sigma):
                d = np.subtract(ws0[w], states[reads[t]], dtype=np.float32)
                e = np.multiply(a, d, dtype=np.float32)
                ws[w] = np.subtract(ws0[w], e, dtype=np.float32)
                states.append(_centre_add(states[-1], e, add))
            out.append((ws, states[-1]))
    return out


def easgd_concurrent_admissible(workers, center, alpha, got_workers, got_center, add="ieee"):
    """Per element: True where (got_workers, got_center) equals, bit for bit (NaNs
    matching NaNs), the result of at least one path of easgd_interleavings --
    the same path for the workers and the centre of that element."""
    def same(u, v):
        u = np.asarray(u, dtype=np.float32)
        v = np.asarray(v, dtype=np.float32)
        return (u.view(np.uint32) == v.view(np.uint32)) | (np.isnan(u) & np.isnan(v))
    ok = np.zeros(np.asarray(center).shape, dtype=bool)
    for ws, c in easgd_interleavings(workers, center, alpha, add):
        m = same(c, got_center)
        for w, g in zip(ws, got_workers):
            m &= same(w, g)
        ok |= m
    return ok
