"""Shared helpers for the -m gpu tests (never imported by the product path)."""

import os

import numpy as np
import torch


def to_dev(arrs, device="cuda:0"):
    return [torch.from_numpy(np.ascontiguousarray(a)).to(device) for a in arrs]


def to_host(ts):
    torch.cuda.synchronize()
    return [t.cpu().numpy() for t in ts]


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


def assert_bitwise(got, want, msg=""):
    got = np.asarray(got, np.float32)
    want = np.asarray(want, np.float32)
    assert got.shape == want.shape, (got.shape, want.shape)
    ok = (bits(got) == bits(want)) | (np.isnan(got) & np.isnan(want))
    if not ok.all():
        i = int(np.argmax(~ok))
        raise AssertionError(f"{msg}: {int((~ok).sum())} of {ok.size} elements differ; first at {i}: "
                             f"got {got[i]!r} ({bits(got)[i]:08x}) want {want[i]!r} ({bits(want)[i]:08x})")


def q11_bound(X):
    """DESIGN.md Q11: 1e-6 * mean_j |x_ij| (fp64)."""
    return 1e-6 * np.mean(np.abs(np.stack(X).astype(np.float64)), axis=0)


def fuzz_cases(k, pmax, n=None):
    """Seeded random multi-process cases for k processes (run by mp_worker.py's
    fuzz mode, checked by test_gpu_multiprocess.py::test_multiprocess_fuzz_bitwise):
    P log-uniform in [1, pmax] (ragged), ASA or ASA16, avg or sum, any staged
    flavour or the runtime's choice, D1-D5, 1-3 calls each a full exchange or a
    bucket with a CTA budget -- or (bsp) two BSP iterations, momentum-SGD step
    fused into the exchange, with or without the momentum exchange."""
    n = int(os.environ.get("TM_MP_FUZZ_CASES", "24")) if n is None else n
    flavours = [None, "reg", "tma", "ws", "tmaws", "oneshot", "ll", "ll2"]
    out = []
    for i in range(n):
        g = np.random.default_rng([1605, 8325, 779, k, i])
        P = max(1, min(pmax, int(np.exp(g.uniform(0.0, np.log(pmax)))) + int(g.integers(0, 4))))
        strategy = ["asa", "asa16"][int(g.integers(0, 2))]
        op = "sum" if g.random() < 0.3 else "avg"
        flavour = flavours[int(g.integers(0, len(flavours)))]
        dist = ["D1", "D2", "D3", "D4", "D5"][int(g.integers(0, 5))]  # D6 overflows a sum
        calls = []
        for _ in range(int(g.integers(1, 4))):
            if P >= 8 and g.random() < 0.5:
                off = int(g.integers(0, P // 4)) * 4
                calls.append((off, int(g.integers(0, P - off + 1)), [0, 1, 3, 16][int(g.integers(0, 4))]))
            else:
                calls.append((0, P, 0))
        bsp = None
        if op == "avg" and g.random() < 0.3:  # a BSP iteration pair instead of the calls
            bsp = dict(mom=bool(g.random() < 0.5), lr=float(np.float32(g.choice([0.01, 0.3]))),
                       mu=float(np.float32(g.choice([0.0, 0.9]))))
        out.append(dict(P=P, strategy=strategy, op=op, flavour=flavour, dist=dist, calls=calls, bsp=bsp))
    return out
