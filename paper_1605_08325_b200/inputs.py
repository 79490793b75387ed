"""Seeded synthetic worker buffers shared by the tests, smoke() and bench.py.

Holds NO arithmetic of the method (no sums, averages, casts): only random draws,
so both the CUDA path and the oracle consume identical bits.  Recipe (DESIGN.md
"Input recipe"):

  seeds  numpy.random.default_rng([1605, 8325, config, dist, rank])
  D1 uniform[-1, 1]
  D2 N(0, 0.01^2)          weight-like; ~0.5% of values in the fp16 subnormal range
  D3 near-equal replicas   w + N(0, 1e-4^2), w ~ N(0, 0.01^2) shared by all ranks
                           (AWAGD after one step)
  D4 N(0, 1e-5^2)          SUBGD-delta-like; mostly fp16 subnormals
  D5 integers in [-256, 256]                  exact-arithmetic cases
  D6 specials: +-0, 65504, 65519.99, 65520, 2^-14, 2^-24, 2^-25 ties, fp32
     subnormals, 1/3, mixed with D1 values

Workload sizes (PAPER Table 3):
  alexnet 60,965,224   googlenet 6,998,552 (main; 13,378,280 with aux)
  vggnet 138,357,544   1M 1,048,576 (tail case 1,000,003)
"""

import numpy as np

WORKLOADS = {
    "1m": 1_048_576,
    "1m_tail": 1_000_003,
    "googlenet": 6_998_552,
    "googlenet_aux": 13_378_280,
    "alexnet": 60_965_224,
    "vggnet": 138_357_544,
}

DISTS = ("D1", "D2", "D3", "D4", "D5", "D6")

_SPECIALS = np.array(
    [0.0, -0.0, 65504.0, -65504.0, 65519.99, 2.0 ** -14, -(2.0 ** -14), 2.0 ** -24,
     2.0 ** -25, -(2.0 ** -25), 3 * 2.0 ** -26, 2.0 ** -25 + 2.0 ** -40, 1e-40, -1e-42,
     1.0 / 3.0, 0.1, 1.0, -1.0, 2048.0, 2047.0, 1.5, 6.1e-5],
    dtype=np.float32)


def _rng(config, dist, rank):
    return np.random.default_rng([1605, 8325, int(config), int(DISTS.index(dist)), int(rank)])


def worker_buffer(P, dist="D1", rank=0, config=0):
    """float32[P] buffer of worker `rank` for distribution `dist`."""
    if dist not in DISTS:
        raise ValueError(dist)
    g = _rng(config, dist, rank)
    if dist == "D1":
        return g.uniform(-1.0, 1.0, P).astype(np.float32)
    if dist == "D2":
        return (g.standard_normal(P, dtype=np.float32) * np.float32(0.01)).astype(np.float32)
    if dist == "D3":
        base = np.random.default_rng([1605, 8325, int(config), 2, 1 << 20])
        w = base.standard_normal(P, dtype=np.float32) * np.float32(0.01)
        return (w + g.standard_normal(P, dtype=np.float32) * np.float32(1e-4)).astype(np.float32)
    if dist == "D4":
        return (g.standard_normal(P, dtype=np.float32) * np.float32(1e-5)).astype(np.float32)
    if dist == "D5":
        return g.integers(-256, 257, P).astype(np.float32)
    # D6: specials sprinkled over uniform values
    x = g.uniform(-1.0, 1.0, P).astype(np.float32)
    if P:
        idx = g.integers(0, P, max(1, P // 4))
        x[idx] = g.choice(_SPECIALS, idx.shape[0]) * g.choice(
            np.array([1.0, -1.0], dtype=np.float32), idx.shape[0])
    return x


def worker_buffers(P, k, dist="D1", config=0):
    """List of k worker buffers."""
    return [worker_buffer(P, dist, r, config) for r in range(k)]


def dyadic_buffers(P, k, config=0, bits=10):
    """Buffers of small dyadic values m * 2^-bits, |m| <= 2^9: every summation order
    is exact for k <= 8, so AR == ASA == the exact mean bitwise."""
    out = []
    for r in range(k):
        g = np.random.default_rng([1605, 8325, int(config), 99, r])
        m = g.integers(-512, 513, P)
        out.append((m.astype(np.float64) * 2.0 ** -bits).astype(np.float32))
    return out
