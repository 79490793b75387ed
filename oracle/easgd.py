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
arithmetic and within one rounding in fp32).  Concurrent (unordered) updates have
no bitwise oracle: "parity unpinned" for bitwise comparison; they are checked by
invariants only.
"""

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
