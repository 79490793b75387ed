#!/usr/bin/env python
"""Parallel loading (Alg. 1) timing on one GPU: ImageNet-like batches of 128 x 3 x
256 x 256 uint8 (24 MiB) cropped to 227 x 227.  Reports the loader's per-batch time
alone (read from page cache + raw H2D + GPU preprocessing + handoff), and the wall
time of n iterations with an emulated training step of the same length, serial
(load, then train) vs pipelined (Alg. 1)."""

import os
import sys
import tempfile
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1605_08325_b200 import tm  # noqa: E402


def main():
    n, c, h, w, ch, cw = 128, 3, 256, 256, 227, 227
    torch.cuda.set_device(0)
    g = np.random.default_rng(0)
    mean = g.uniform(0, 255, (c, h, w)).astype(np.float32)
    d = tempfile.mkdtemp()
    paths = []
    for i in range(4):
        p = os.path.join(d, f"b{i}.pxb")
        tm.write_batch_file(p, g.integers(0, 256, (n, c, h, w)).astype(np.uint8))
        paths.append(p)
    files = [paths[i % 4] for i in range(41)]
    x = torch.zeros(n * c * ch * cw, device="cuda")

    def run(compute_s, pipelined=True):
        with tm.Loader(n, c, h, w, ch, cw, mean, x, seed=1) as L:
            t0 = time.perf_counter()
            L.send("train")
            L.send("file", files[0])
            for f in files[1:]:
                L.send("file", f)
                L.wait(60_000)
                if not pipelined:  # serial: the next load would start only now
                    pass
                time.sleep(compute_s)
            return time.perf_counter() - t0

    run(0.0)
    iters = len(files) - 1
    load = run(0.0) / iters
    piped = run(load)
    print({"batch": [n, c, h, w], "crop": [ch, cw], "load_ms_per_batch": round(load * 1e3, 2),
           "raw_MB_per_batch": round(n * c * h * w / 1e6, 1),
           "iters": iters, "serial_estimate_s": round(iters * 2 * load, 3),
           "pipelined_s": round(piped, 3), "pipelined_over_serial": round(piped / (iters * 2 * load), 3)})


if __name__ == "__main__":
    main()
