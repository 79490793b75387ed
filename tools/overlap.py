#!/usr/bin/env python
"""Overlapping the exchange with backward.

k = 8 workers' AlexNet-sized parameter vectors on one GPU (single-process group).
"Backward" is emulated layer by layer, last layer first, as bf16 GEMMs whose
FLOPs follow AlexNet's per-layer backward cost for a 128-image batch per worker
(2 x forward MACs x 2 FLOP/MAC x 128 x 8 workers).  Two schedules:

  serial     all layers' GEMMs, then one tm_exchange_group of the whole buffer
  overlapped after each layer's GEMM an event; a second stream waits for it and
             exchanges that layer's bucket with tm_exchange_group_range

Prints ms per iteration of each schedule (CUDA events, median of 10 after 3
warm-ups) and the exchange alone.  Run with TM_DIRECT_LDG=1 to use the register
kernel, which leaves shared memory free for the GEMMs' CTAs.

    python tools/overlap.py [--budgets 0,8,16,32,64] [--priority]

--budgets: CTA budgets of the bucket exchanges (tm_set_range_ctas; 0 = none,
the full persistent grid); --priority: the exchange stream at high priority,
so its CTAs are dispatched as soon as a GEMM CTA retires.
"""

import argparse
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1605_08325_b200 import tm  # noqa: E402

# (name, W+b parameters, forward MACs per image) -- AlexNet, 2-group
LAYERS = [("conv1", 34_944, 105e6), ("conv2", 307_456, 224e6), ("conv3", 885_120, 150e6),
          ("conv4", 663_936, 112e6), ("conv5", 442_624, 75e6), ("fc6", 37_752_832, 38e6),
          ("fc7", 16_781_312, 17e6), ("fc8", 4_097_000, 4e6)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--budgets", default="0,8,16,32,64")
    ap.add_argument("--priority", action="store_true")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    k, batch = 8, 128
    P = sum(n for _, n, _ in LAYERS)
    offs, o = [], 0
    for _, n, _ in LAYERS:
        offs.append(o)
        o += n
    bufs = [torch.randn(P, device="cuda") * 0.01 for _ in range(k)]
    gemms = []
    for _, _, macs in LAYERS:
        flops = 2 * macs * 2 * batch * k  # backward ~ 2x forward, 2 FLOP per MAC
        n = max(256, int(round((flops / 2) ** (1 / 3) / 128)) * 128)
        a = torch.randn(n, n, device="cuda", dtype=torch.bfloat16)
        gemms.append((a, torch.randn(n, n, device="cuda", dtype=torch.bfloat16)))
    sa = torch.cuda.Stream()
    sb = torch.cuda.Stream(priority=-1) if args.priority else torch.cuda.Stream()
    ex = tm.Exchanger(P, "asa16", size=k, nlocal=k)

    def backward(stream, events=None):
        with torch.cuda.stream(stream):
            for li in reversed(range(len(LAYERS))):
                a, b = gemms[li]
                torch.matmul(a, b)
                if events is not None:
                    events[li].record(stream)

    def serial():
        backward(sa)
        ex.exchange(bufs, sa)

    def overlapped():
        evs = [torch.cuda.Event() for _ in LAYERS]
        backward(sa, evs)
        for li in reversed(range(len(LAYERS))):
            sb.wait_event(evs[li])
            ex.exchange_range(bufs, offs[li], LAYERS[li][1], sb)

    def exchange_only():
        ex.exchange(bufs, sa)

    def backward_only():
        backward(sa)

    def timed(fn):
        out = []
        for it in range(13):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(torch.cuda.current_stream())
            sa.wait_stream(torch.cuda.current_stream())
            sb.wait_stream(torch.cuda.current_stream())
            fn()
            torch.cuda.current_stream().wait_stream(sa)
            torch.cuda.current_stream().wait_stream(sb)
            e1.record(torch.cuda.current_stream())
            torch.cuda.synchronize()
            if it >= 3:
                out.append(e0.elapsed_time(e1))
        return statistics.median(out)

    def buckets_only():
        for li in reversed(range(len(LAYERS))):
            ex.exchange_range(bufs, offs[li], LAYERS[li][1], sb)

    res = {name: timed(fn) for name, fn in (("backward_only", backward_only), ("exchange_only", exchange_only),
                                            ("serial", serial))}
    for b in [int(v) for v in args.budgets.split(",")]:
        tm.tm_set_range_ctas(b)
        res[f"buckets_only_budget{b}"] = timed(buckets_only)
        res[f"overlapped_budget{b}"] = timed(overlapped)
    tm.tm_set_range_ctas(0)
    code, _ = ex.status()
    ex.finalize()
    kern = "register" if os.environ.get("TM_DIRECT_LDG") == "1" else "tma"
    best = min((v, n) for n, v in res.items() if n.startswith("overlapped"))
    print(json.dumps({"direct_kernel": kern, "priority_stream": args.priority,
                      **{k_: round(v, 3) for k_, v in res.items()}, "status": code,
                      "best_overlapped": best[1], "hidden_ms": round(res["serial"] - best[0], 3)}))


if __name__ == "__main__":
    main()
