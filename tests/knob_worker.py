#!/usr/bin/env python
"""One scenario of tests/test_gpu_knobs.py in a fresh process, so that the
library's diagnostics knobs that are read once per process (TM_L2_HINT,
TM_BSP_TILE, TM_ROUND_STATIC, ...) take the value in this process's
environment.  Every scenario compares the GPU result with the oracle bit for
bit; exit code 0 = bitwise, 3 = mismatch.

    python tests/knob_worker.py direct|direct_small_k|bsp|round|oneshot|ranges|staged
"""

import os
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from oracle import exchange as ox  # noqa: E402  (test infrastructure)
from oracle.bsp import bsp_iteration  # noqa: E402
from oracle.easgd import easgd_sequence  # noqa: E402
from paper_1605_08325_b200 import tm  # noqa: E402
from paper_1605_08325_b200.inputs import worker_buffer, worker_buffers  # noqa: E402


def same(a, b):
    return np.array_equal(np.asarray(a, np.float32).view(np.uint32), np.asarray(b, np.float32).view(np.uint32))


def dev(xs):
    return [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in xs]


def host(ts):
    torch.cuda.synchronize()
    return [t.cpu().numpy() for t in ts]


def check_all(got, want, what):
    for r, (g, w) in enumerate(zip(got, want)):
        if not same(g, w):
            bad = np.flatnonzero(np.asarray(g, np.float32).view(np.uint32) != np.asarray(w, np.float32).view(np.uint32))
            print(f"MISMATCH {what} rank {r}: {bad.size} elements, first {bad[0]}")
            sys.exit(3)


def exchange_scenario(k, P, strategies, path, ranges=None, config=170):
    for strategy in strategies:
        X = worker_buffers(P, k, "D2", config=config)
        bufs = dev(X)
        with tm.Exchanger(P, strategy, size=k, nlocal=k, path=path) as ex:
            for _ in range(2):
                if ranges is None:
                    ex.exchange(bufs)
                else:
                    for off, cnt in ranges:
                        ex.exchange_range(bufs, off, cnt)
            code, _ = ex.status()
        assert code == tm.TM_OK, code
        want = X
        for _ in range(2):
            want = ox.exchange(want, strategy)
        check_all(host(bufs), want, f"{strategy} {path} k={k} P={P}")


def main():
    torch.cuda.set_device(0)
    what = sys.argv[1]
    if what == "direct":  # k * P above the register-kernel threshold: the TMA direct kernel
        exchange_scenario(8, 1_500_007, ("asa16", "asa"), "direct")
    elif what == "direct_small_k":  # k <= 4 on the TMA direct kernel (its own TM_TMA_CFG variants)
        exchange_scenario(2, 5_000_011, ("asa16",), "direct")
        exchange_scenario(4, 3_000_007, ("asa16", "asa"), "direct")
    elif what == "bsp":  # the fused BSP kernel on the TMA engine (k * P > 4 Mi)
        k, P, lr, mu = 8, 1_000_003, 0.01, 0.9
        W = worker_buffers(P, k, "D2", config=171)
        V = worker_buffers(P, k, "D4", config=172)
        G = worker_buffers(P, k, "D2", config=173)
        Wd, Vd, Gd = dev(W), dev(V), dev(G)
        with tm.Exchanger(P, "asa16", size=k, nlocal=k, path="direct") as ex:
            ex.bsp_step(Wd, Vd, Gd, lr, mu, exchange_momentum=True)
            code, _ = ex.status()
        assert code == tm.TM_OK, code
        ww, vv = bsp_iteration(W, V, G, lr, mu, "asa16", exchange_momentum=True)
        check_all(host(Wd), ww, "bsp w")
        check_all(host(Vd), vv, "bsp v")
    elif what == "round":  # a fused EASGD round of 8 distinct workers on the TMA engine
        n, alpha, order = 3_000_001, np.float32(0.3), [5, 2, 7, 0, 1, 6, 3, 4]
        W = [worker_buffer(n, "D1", r, config=174) for r in range(8)]
        c = worker_buffer(n, "D1", 99, config=174)
        Wd, cd = dev(W), dev([c])[0]
        tm.tm_easgd_round(Wd, order, cd, float(alpha))
        ww, wc = easgd_sequence(W, c, alpha, order)
        check_all(host(Wd), ww, "round workers")
        check_all(host([cd]), [wc], "round centre")
    elif what == "oneshot":
        exchange_scenario(4, 200_003, ("asa16", "asa"), "staged")
    elif what == "ranges":  # TM_RANGE_CTAS at init: every bucket on a CTA budget
        P = 900_007
        b1, b2 = P // 3 // 4 * 4, 2 * P // 3 // 4 * 4
        rg = ((b2, P - b2), (b1, b2 - b1), (0, b1))
        exchange_scenario(4, P, ("asa16",), "staged", ranges=rg)
        exchange_scenario(4, P, ("asa16",), "direct", ranges=rg)
    elif what == "staged":
        exchange_scenario(3, 100_003, ("asa16", "asa"), "staged")
    else:
        raise SystemExit(f"unknown scenario {what}")
    print("OK", what)


if __name__ == "__main__":
    main()
