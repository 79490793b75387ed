#!/usr/bin/env python
"""Latency of the BSP step (direct path, momentum exchanged) and of an EASGD
round (8 workers, arrival order) at small sizes, one GPU, 64 calls per CUDA
graph; run once plain and once with TM_DIRECT_LDG=1 (register kernels) to
place the TMA / register threshold.  One JSON line per size."""
import json
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
    k = 8
    sizes = [int(v) for v in os.environ.get("TM_SMALL_SIZES", "4096,32768,131072,524288,1048576,2097152").split(",")]
    for P in sizes:
        W = [torch.randn(P, device="cuda") * 0.01 for _ in range(k)]
        V = [torch.zeros(P, device="cuda") for _ in range(k)]
        G = [torch.randn(P, device="cuda") * 0.01 for _ in range(k)]
        with tm.Exchanger(P, "asa16", size=k, nlocal=k, path="direct") as ex:
            bsp = timeit(lambda: ex.bsp_step(W, V, G, 0.01, 0.9, exchange_momentum=True), graph=True) * 1e3
        c = torch.randn(P, device="cuda") * 0.01
        rnd = timeit(lambda: tm.tm_easgd_round(W, list(range(k)), c, 0.5 / k), graph=True) * 1e3
        print(json.dumps({"P": P, "k": k, "ldg": os.environ.get("TM_DIRECT_LDG") == "1",
                          "bsp_us": bsp, "easgd_round_us": rnd}), flush=True)
        del W, V, G, c
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
