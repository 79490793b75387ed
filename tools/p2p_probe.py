#!/usr/bin/env python
"""Peer-to-peer copy bandwidth between GPU pairs (copy engines, through torch's
cross-device copy): the per-direction NVLink figure the staged kernels' a4 / a6
phases and the TM_AG_CE allgather are bounded by (770 GB/s measured on this pool
per B200_PROFILING.md; 900 nominal).  Needs >= 2 GPUs; one JSON line per pair.

    python tools/p2p_probe.py [--mb 1024] [--pairs 0-1,0-7]
"""

import argparse
import json

import torch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=int, default=1024)
    ap.add_argument("--pairs", default=None)
    a = ap.parse_args()
    n = torch.cuda.device_count()
    if n < 2:
        print(json.dumps({"skipped": f"{n} GPU(s) visible; peer copies need 2"}))
        return
    pairs = ([tuple(int(v) for v in p.split("-")) for p in a.pairs.split(",")] if a.pairs
             else [(0, j) for j in range(1, n)])
    nbytes = a.mb << 20
    for i, j in pairs:
        src = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{i}")
        dst = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{j}")
        can = torch.cuda.can_device_access_peer(j, i)
        with torch.cuda.device(j):
            for _ in range(3):
                dst.copy_(src, non_blocking=True)
            torch.cuda.synchronize(j)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            reps = 10
            for _ in range(reps):
                dst.copy_(src, non_blocking=True)
            e1.record()
            torch.cuda.synchronize(j)
            ms = e0.elapsed_time(e1) / reps
        print(json.dumps({"src": i, "dst": j, "peer_access": bool(can), "bytes": nbytes,
                          "ms": ms, "GBps": nbytes / (ms * 1e-3) / 1e9}), flush=True)


if __name__ == "__main__":
    main()
