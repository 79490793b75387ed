#!/usr/bin/env python
"""Small-message latency of one exchange (CUDA-graph replay, 64 exchanges per
graph), one GPU, k ranks in one process: the direct path and every staged
flavour (TM_STAGED_KERNEL is read at init), plus the default flavour chosen by
the segment length.  One JSON line per measurement.

    python tools/latency.py [--k 2,4,8] [--P 2048,...] [--strategy asa16]
"""

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

from paper_1605_08325_b200 import tm  # noqa: E402
from sweep import timeit  # noqa: E402

NAMES = {0: "reg", 1: "tma", 2: "ws", 3: "tmaws", 4: "oneshot", 5: "ll", 6: "ll2"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--k", default="2,4,8")
    ap.add_argument("--P", default="2048,8192,32768,65536,131072,262144,524288,1048576,2097152,4194304")
    ap.add_argument("--strategy", default="asa16")
    ap.add_argument("--flavours", default="default,oneshot,reg,tma,tmaws,ws")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    for P in [int(v) for v in a.P.split(",")]:
        for k in [int(v) for v in a.k.split(",")]:
            bufs = [torch.randn(P, device="cuda") for _ in range(k)]
            variants = [("direct", None)] + [("staged", f) for f in a.flavours.split(",") if f]
            for path, fl in variants:
                os.environ.pop("TM_STAGED_KERNEL", None)
                if fl and fl != "default":
                    os.environ["TM_STAGED_KERNEL"] = fl
                with tm.Exchanger(P, a.strategy, size=k, nlocal=k, path=path) as ex:
                    us = timeit(lambda: ex.exchange(bufs), graph=True) * 1e3
                    lay = ex.layout()
                os.environ.pop("TM_STAGED_KERNEL", None)
                print(json.dumps({"P": P, "k": k, "strategy": a.strategy, "path": path,
                                  "flavour": (fl if path == "staged" else None),
                                  "kernel": NAMES[lay["staged_kernel"]] if path == "staged" else "direct",
                                  "L": lay["seg_len"], "C": lay["ctas_per_rank"], "us": us}), flush=True)
            del bufs
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
