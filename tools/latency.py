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
    # staged: every kernel flavour (TM_STAGED_KERNEL is read at init)
    variants = [("direct", None), ("staged", "tma"), ("staged", "tmaws"), ("staged", "ws"), ("staged", "reg")]
    for P in (2048, 16384, 65536, 262144, 1 << 20, 1 << 22):
        for k in (2, 8):
            for path, fl in variants:
                if fl:
                    os.environ["TM_STAGED_KERNEL"] = fl
                bufs = [torch.randn(P, device="cuda") for _ in range(k)]
                with tm.Exchanger(P, "asa16", size=k, nlocal=k, path=path) as ex:
                    us = timeit(lambda: ex.exchange(bufs), graph=True) * 1e3
                    lay = ex.layout()
                os.environ.pop("TM_STAGED_KERNEL", None)
                name = path if not fl else f"{path}/{fl}"
                print(f"P={P:8d} k={k} {name:11s} C={lay['ctas_per_rank']:4d} {us:8.2f} us", flush=True)


if __name__ == "__main__":
    main()
