#!/usr/bin/env python
"""Small-message latency of one exchange (CUDA-graph replay), one GPU."""

import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

from paper_1605_08325_b200 import tm  # noqa: E402
from sweep import timeit  # noqa: E402


def main():
    torch.cuda.set_device(0)
    for P in (2048, 65536, 1 << 20):
        for k in (2, 8):
            for path in ("direct", "staged"):
                bufs = [torch.randn(P, device="cuda") for _ in range(k)]
                with tm.Exchanger(P, "asa16", size=k, nlocal=k, path=path) as ex:
                    us = timeit(lambda: ex.exchange(bufs), graph=True) * 1e3
                    lay = ex.layout()
                print(f"P={P:8d} k={k} {path:7s} C={lay['ctas_per_rank']:4d} {us:8.2f} us", flush=True)


if __name__ == "__main__":
    main()
