#!/usr/bin/env python
"""A few calls of one library entry point at AlexNet size, k = 8 ranks on one GPU
(a short target for ncu captures; no timing).

    python tools/one_call.py exchange-direct|exchange-staged|bsp-direct|bsp-staged|bsp-staged-mom|easgd-round [n]

TM_ONE_CALL_P / TM_ONE_CALL_K override the size and rank count (e.g. a small P
for the one-shot kernel).
"""

import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1605_08325_b200 import tm  # noqa: E402

P = int(os.environ.get("TM_ONE_CALL_P", "60965224"))
K = int(os.environ.get("TM_ONE_CALL_K", "8"))


def main():
    what = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    torch.cuda.set_device(0)
    g = torch.Generator(device="cuda").manual_seed(1)
    W = [torch.randn(P, device="cuda", generator=g) * 0.01 for _ in range(K)]
    if what.startswith("exchange"):
        with tm.Exchanger(P, "asa16", size=K, nlocal=K, path=what.split("-")[1]) as ex:
            for _ in range(n):
                ex.exchange(W)
    elif what.startswith("bsp"):
        V = [torch.zeros(P, device="cuda") for _ in range(K)]
        G = [torch.randn(P, device="cuda", generator=g) * 0.01 for _ in range(K)]
        with tm.Exchanger(P, "asa16", size=K, nlocal=K, path=what.split("-")[1]) as ex:
            for _ in range(n):
                ex.bsp_step(W, V, G, 0.01, 0.9, exchange_momentum=what.endswith("-mom"))
    elif what == "easgd-round":
        c = torch.randn(P, device="cuda", generator=g) * 0.01
        for _ in range(n):
            tm.tm_easgd_round(W, list(range(K)), c, 0.5 / K)
    else:
        raise SystemExit(f"unknown call {what}")
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
