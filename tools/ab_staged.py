#!/usr/bin/env python
"""A/B helper: staged-path timings (CUDA-graph replay) of a few configs in this
process's environment (e.g. TM_TMA_SUBREADY=0/1, TM_STAGED_KERNEL=...).
One JSON line per config."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from sweep import exchange_row, peak  # noqa: E402

CONFIGS = [(60_965_224, 8), (60_965_224, 4), (60_965_224, 2), (6_998_552, 8), (2_097_152, 8), (8_388_608, 8)]


def main():
    torch.cuda.set_device(0)
    pk = peak()
    for P, k in CONFIGS:
        r = exchange_row(P, k, "asa16", "staged", pk)
        r["env"] = {k_: v for k_, v in os.environ.items() if k_.startswith("TM_")}
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
