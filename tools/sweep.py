#!/usr/bin/env python
"""One-GPU timing sweep over the BASELINE.json configs:

  config 2  GoogLeNet 6,998,552      ASA, ASA16        k = 2, 4, 8   direct + staged
  config 3  AlexNet   60,965,224     AR, ASA, ASA16    k = 2, 4, 8   direct + staged
  config 4  EASGD 8 workers + centre, AlexNet size, alpha = 0.5/8:
            8 serial exclusive updates / one fused arrival-order round /
            8 concurrent updates (red.add) from 8 streams
  config 5  message-size sweep 64 KB .. 1 GB (fp32 bytes per rank), ASA16, k = 2, 4, 8

Every call is captured once in a CUDA graph and replayed (no host launch
overhead in the numbers).  All ranks of an exchange live on this one GPU (single-process group), so every
number is HBM-bound; the roofline is the measured HBM copy bandwidth.  Inputs are
N(0, 0.01^2) drawn on the device (timing only; parity lives in tests/).
Writes JSON lines to stdout and a markdown table to --md.
"""

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1605_08325_b200 import tm  # noqa: E402

ALEXNET, GOOGLENET = 60_965_224, 6_998_552


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def timeit(fn, min_ms=60.0, warmup=5, graph=False):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    inner = 1
    if graph:  # replay a captured call: no host launch overhead in the timing
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        # short calls: capture `inner` back-to-back calls per graph, so the GPU is
        # never starved by the host's replay rate (~2 us per replay)
        inner = 64 if e0.elapsed_time(e1) < 0.2 else 1
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(inner):
                fn()
        fn = g.replay
        fn()
        torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    one = max(e0.elapsed_time(e1), 1e-3)
    n = max(5, min(2000, int(min_ms / one)))
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (n * inner)


def hbm_bytes(strategy, P, k, path):
    if path == "direct" or strategy == "ar":
        return 8.0 * P * k
    return (14 + 2.0 / k) * P * k if strategy == "asa16" else (20 + 4.0 / k) * P * k


def exchange_row(P, k, strategy, path, pk):
    g = torch.Generator(device="cuda").manual_seed(1605)
    bufs = [torch.randn(P, device="cuda", generator=g) * 0.01 for _ in range(k)]
    with tm.Exchanger(P, strategy, size=k, nlocal=k, path=path) as ex:
        ms = timeit(lambda: ex.exchange(bufs), graph=True)
        code, _ = ex.status()
    alg = hbm_bytes(strategy, P, k, path)
    row = {"P": P, "k": k, "strategy": strategy, "path": path if strategy != "ar" else "direct",
           "us": ms * 1e3, "algbw_GBps": 4.0 * P * k / (ms * 1e-3) / 1e9,
           "hbm_GBps": alg / (ms * 1e-3) / 1e9, "frac": alg / (ms * 1e-3) / 1e9 / pk, "status": code,
           "l2_resident": 4.0 * P * k <= 100e6}
    del bufs
    torch.cuda.empty_cache()
    return row


def easgd_rows(P, nw, alpha, pk):
    g = torch.Generator(device="cuda").manual_seed(8325)
    W = [torch.randn(P, device="cuda", generator=g) * 0.01 for _ in range(nw)]
    c = torch.randn(P, device="cuda", generator=g) * 0.01
    rows = []

    def serial():
        for w in W:
            tm.tm_easgd_update_ex(w, c, alpha)
    ms = timeit(serial, graph=True)
    rows.append({"mode": f"{nw} serial exclusive updates", "us": ms * 1e3,
                 "hbm_GBps": 16.0 * P * nw / (ms * 1e-3) / 1e9})
    order = list(range(nw))
    ms = timeit(lambda: tm.tm_easgd_round(W, order, c, alpha), graph=True)
    rows.append({"mode": f"fused round, arrival order of {nw}", "us": ms * 1e3,
                 "hbm_GBps": (8.0 * P * nw + 8.0 * P) / (ms * 1e-3) / 1e9})
    streams = [torch.cuda.Stream() for _ in range(nw)]

    def concurrent(mode):
        cur = torch.cuda.current_stream()
        ev = torch.cuda.Event()
        ev.record(cur)
        for w, s in zip(W, streams):
            s.wait_event(ev)
            tm.tm_easgd_update_ex(w, c, alpha, concurrent=mode, stream=s)
        for s in streams:
            cur.wait_stream(s)
    ms = timeit(lambda: concurrent(1))
    rows.append({"mode": f"{nw} concurrent updates (red.add, {nw} streams)", "us": ms * 1e3,
                 "hbm_GBps": 16.0 * P * nw / (ms * 1e-3) / 1e9})
    ms = timeit(lambda: concurrent("exact"))
    rows.append({"mode": f"{nw} concurrent updates (exact: CAS-loop IEEE add, 128-bit CAS, {nw} streams)",
                 "us": ms * 1e3, "hbm_GBps": 16.0 * P * nw / (ms * 1e-3) / 1e9})
    os.environ["TM_EASGD_CAS128"] = "0"  # the 32-bit CAS per element (a centre on a peer GPU)
    ms = timeit(lambda: concurrent("exact"))
    del os.environ["TM_EASGD_CAS128"]
    rows.append({"mode": f"{nw} concurrent updates (exact: CAS-loop IEEE add, 32-bit CAS, {nw} streams)",
                 "us": ms * 1e3, "hbm_GBps": 16.0 * P * nw / (ms * 1e-3) / 1e9})
    del c
    with tm.Exchanger(P, "easgd", size=nw, nlocal=nw) as ex:
        for sidx in range(nw):
            ex.center_shard(sidx).normal_(0, 0.01)

        def sharded():
            for w in W:
                tm.tm_easgd_update_sharded(w, alpha)
        ms = timeit(sharded, graph=True)
        rows.append({"mode": f"{nw} serial updates, centre sharded by segment over {nw} ranks",
                     "us": ms * 1e3, "hbm_GBps": 16.0 * P * nw / (ms * 1e-3) / 1e9})
    for r in rows:
        r["frac"] = r["hbm_GBps"] / pk
        r["P"] = P
    return rows


def bsp_rows(P, k, pk):
    """NEXT-1: momentum-SGD step + exchange of k workers, fused in one pass (direct
    path) vs the library's unfused sequence (SGD kernel per worker, then the
    direct exchange; TM_BSP_UNFUSED=1), with and without momentum exchange."""
    g = torch.Generator(device="cuda").manual_seed(77)
    W = [torch.randn(P, device="cuda", generator=g) * 0.01 for _ in range(k)]
    V = [torch.zeros(P, device="cuda") for _ in range(k)]
    G = [torch.randn(P, device="cuda", generator=g) * 0.01 for _ in range(k)]
    rows = []
    for path in ("direct", "staged"):
        for mom in (False, True):
            for fused in (True, False):
                os.environ["TM_BSP_UNFUSED"] = "0" if fused else "1"
                with tm.Exchanger(P, "asa16", size=k, nlocal=k, path=path) as ex:
                    ms = timeit(lambda: ex.bsp_step(W, V, G, 0.01, 0.9, exchange_momentum=mom), graph=True)
                # irreducible: read w, v, g + write w, v = 20 B per element per worker
                alg = 20.0 * P * k
                how = ("fused one pass" if path == "direct" else "step fused into the pre-cast") if fused \
                    else "SGD pass + exchange pass(es)"
                rows.append({"mode": f"{path}: {how}{', momentum exchanged' if mom else ''}",
                             "us": ms * 1e3, "hbm_GBps": alg / (ms * 1e-3) / 1e9,
                             "frac": alg / (ms * 1e-3) / 1e9 / pk, "P": P, "k": k})
    os.environ.pop("TM_BSP_UNFUSED", None)
    return rows


def allgather_rows(P, k, pk):
    """a6 modes on the staged path (tm_allgather): the fused SM pull vs the copy
    engines + widen kernel, every staged flavour, ASA16."""
    rows = []
    for fl in ("tma", "tmaws", "ws", "reg"):
        for ag in ("sm", "ce"):
            os.environ["TM_STAGED_KERNEL"] = fl
            g = torch.Generator(device="cuda").manual_seed(1605)
            bufs = [torch.randn(P, device="cuda", generator=g) * 0.01 for _ in range(k)]
            with tm.Exchanger(P, "asa16", size=k, nlocal=k, path="staged", allgather=ag) as ex:
                ms = timeit(lambda: ex.exchange(bufs), graph=True)
            alg = hbm_bytes("asa16", P, k, "staged")
            rows.append({"mode": f"staged/{fl} allgather={ag}", "us": ms * 1e3,
                         "hbm_GBps": alg / (ms * 1e-3) / 1e9, "frac": alg / (ms * 1e-3) / 1e9 / pk,
                         "P": P, "k": k})
            del bufs
            torch.cuda.empty_cache()
    os.environ.pop("TM_STAGED_KERNEL", None)
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--md", default=None)
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--only", choices=["bsp", "easgd", "ag"], default=None,
                    help="time only the BSP rows, the EASGD (config 4) rows or the allgather modes")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    pk = peak()
    if a.only:
        rows = {"bsp": lambda: bsp_rows(ALEXNET, 8, pk), "easgd": lambda: easgd_rows(ALEXNET, 8, 0.5 / 8, pk),
                "ag": lambda: allgather_rows(ALEXNET, 8, pk)}[a.only]()
        for r in rows:
            print(json.dumps({"config": "config4" if a.only == "easgd" else a.only, **r}))
        return
    out = {"config2": [], "config3": [], "config4": [], "config5": [], "bsp": []}
    ks = (2, 4, 8)
    for strategy in ("asa", "asa16"):
        for k in ks:
            for path in ("direct", "staged"):
                out["config2"].append(exchange_row(GOOGLENET, k, strategy, path, pk))
    for strategy in ("ar", "asa", "asa16"):
        for k in ks:
            for path in (("direct",) if strategy == "ar" else ("direct", "staged")):
                out["config3"].append(exchange_row(ALEXNET, k, strategy, path, pk))
    out["config4"] = easgd_rows(ALEXNET, 8, 0.5 / 8, pk)
    out["bsp"] = bsp_rows(ALEXNET, 8, pk)
    sizes = [1 << e for e in range(16, 31, 2 if a.quick else 1)]
    for nbytes in sizes:
        P = nbytes // 4
        for k in ks:
            if P * k * 4 > 24 * (1 << 30):
                continue
            for path in ("direct", "staged"):
                out["config5"].append(exchange_row(P, k, "asa16", path, pk))
    for key, rows in out.items():
        for r in rows:
            print(json.dumps({"config": key, **r}))
    if a.md:
        with open(a.md, "w") as f:
            f.write(f"# One-GPU sweep (measured HBM peak {pk:.0f} GB/s)\n\n")
            f.write("frac = algorithmic HBM bytes / time / peak. Direct path: 8 B per element "
                    "per rank; staged: (14 + 2/k) B (ASA16), (20 + 4/k) B (ASA). (L2): the k input "
                    "buffers fit in the 126 MB L2 and are re-read from it between replays, so frac > 1 "
                    "there is an L2 effect, not HBM bandwidth; small sizes are latency-bound.\n\n")
            for key in ("config2", "config3", "config5"):
                f.write(f"## {key}\n\n| P | k | strategy | path | µs | algbw GB/s | HBM GB/s | frac |\n"
                        "|---|---|---|---|---|---|---|---|\n")
                for r in out[key]:
                    f.write(f"| {r['P']:,}{' (L2)' if r['l2_resident'] else ''} | {r['k']} | {r['strategy']} | "
                            f"{r['path']} | {r['us']:.1f} | "
                            f"{r['algbw_GBps']:.0f} | {r['hbm_GBps']:.0f} | {r['frac']:.3f} |\n")
                f.write("\n")
            f.write("## config4 (EASGD, 8 workers + centre, P = 60,965,224, alpha = 0.5/8)\n\n"
                    "| mode | µs | HBM GB/s | frac |\n|---|---|---|---|\n")
            for r in out["config4"]:
                f.write(f"| {r['mode']} | {r['us']:.1f} | {r['hbm_GBps']:.0f} | {r['frac']:.3f} |\n")
            f.write("\n## BSP iteration (SGD step + exchange), AlexNet, k = 8, ASA16 "
                    "(HBM GB/s counts the fused pass's 20 B per element per worker for both rows)\n\n"
                    "| mode | µs | HBM GB/s | frac |\n|---|---|---|---|\n")
            for r in out["bsp"]:
                f.write(f"| {r['mode']} | {r['us']:.1f} | {r['hbm_GBps']:.0f} | {r['frac']:.3f} |\n")


if __name__ == "__main__":
    main()
