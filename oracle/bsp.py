"""One BSP iteration's update + combine: momentum SGD then the exchange.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Paper anchors: PAPER.md L195-212 (Sec. 3.1: each worker "performs SGD" on its
mini-batch, then parameters are exchanged); L373-384 (Sec. 4: AWAGD averages the
weights after gradient descent; momentum is among the exchanged parameters,
L373-376, and Ding14 exchanges "both weights and momentum", L160-164).  The paper
does not print the SGD update; SPEC.md L280 gives it:

    velocity <- mu * velocity - lr * grad;   weights <- weights + velocity

Here each operation is one fp32 rounding, no FMA:
    v' = fl(fl(mu * v) - fl(lr * g));   w' = fl(w + v')
then the k workers' w' are averaged with the exchange strategy (oracle/exchange.py),
and, if exchange_momentum, the v' too.

Parity status: sgd_step and bsp_iteration are pinned (tests/test_oracle_bsp.py:
SPEC L283-285 examples, exact-rational brute force of each rounding, composition
with the pinned exchange oracle).
"""

import numpy as np

from .exchange import exchange


def sgd_step(w, v, g, lr, mu):
    """Momentum SGD, one fp32 op per step.  Returns (w', v')."""
    w = np.asarray(w, dtype=np.float32)
    v = np.asarray(v, dtype=np.float32)
    g = np.asarray(g, dtype=np.float32)
    mv = np.multiply(np.float32(mu), v, dtype=np.float32)
    lg = np.multiply(np.float32(lr), g, dtype=np.float32)
    v_new = np.subtract(mv, lg, dtype=np.float32)
    w_new = np.add(w, v_new, dtype=np.float32)
    return w_new, v_new


def bsp_iteration(W, V, G, lr, mu, strategy, exchange_momentum=False):
    """Every worker j takes its SGD step, then the weights (and optionally the
    velocities) are averaged across workers with `strategy`.  Returns (W', V')."""
    steps = [sgd_step(w, v, g, lr, mu) for w, v, g in zip(W, V, G)]
    W1 = [s[0] for s in steps]
    V1 = [s[1] for s in steps]
    W2 = exchange(W1, strategy)
    V2 = exchange(V1, strategy) if exchange_momentum else V1
    return W2, V2
