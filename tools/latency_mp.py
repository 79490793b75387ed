#!/usr/bin/env python
"""Latency of the multi-process exchange: k processes (one rank each, CUDA IPC
peer mappings, system-scope flags) on one GPU, run concurrently under CUDA MPS
(TM_PROCS_PER_GPU=k gives each process 1/k of the co-resident CTAs) -- or, on a
multi-GPU box, one process per GPU over NVLink (config 5's message-size sweep,
with --nccl for NCCL's allreduce of the same buffer beside it).  Each
process captures 64 back-to-back exchanges in a CUDA graph and replays it;
time per exchange = max over ranks.  Launched by torchrun (gloo plumbing):

    TM_PROCS_PER_GPU=8 torchrun --nproc-per-node 8 tools/latency_mp.py [--P ...] [--flavours ...]
"""

import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1605_08325_b200 import tm  # noqa: E402

NAMES = {0: "reg", 1: "tma", 2: "ws", 3: "tmaws", 4: "oneshot", 5: "ll", 6: "ll2"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--P", default="2048,8192,32768,65536,131072,262144,524288,1048576,2097152")
    ap.add_argument("--strategy", default="asa16")
    ap.add_argument("--flavours", default="default,oneshot,reg,tma,tmaws")
    ap.add_argument("--inner", type=int, default=64)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--nccl", action="store_true",
                    help="also time torch.distributed.all_reduce (NCCL) of the same buffer (config 5)")
    a = ap.parse_args()
    rank, k = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if torch.cuda.device_count() < k:  # ranks share a GPU: NCCL needs a host id per rank
        os.environ.setdefault("NCCL_HOSTID", f"tm-lat-rank-{rank}")
        os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")
        os.environ.setdefault("NCCL_IB_DISABLE", "1")
    dist.init_process_group("gloo")
    nccl_pg = dist.new_group(backend="nccl") if a.nccl else None
    for P in [int(v) for v in a.P.split(",")]:
        x = torch.randn(P, device="cuda") * 0.01
        nccl_us = None
        if nccl_pg is not None:  # NCCL's fp32 allreduce of the same P floats, max over ranks
            y = x.clone()
            for _ in range(3):
                dist.all_reduce(y, group=nccl_pg)
            torch.cuda.synchronize()
            dist.barrier()
            n0, n1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            n0.record()
            for _ in range(a.reps):
                dist.all_reduce(y, group=nccl_pg)
            n1.record()
            torch.cuda.synchronize()
            tn = torch.tensor([n0.elapsed_time(n1) * 1e3 / a.reps], dtype=torch.float64)
            dist.all_reduce(tn, op=dist.ReduceOp.MAX)
            nccl_us = float(tn.item())
            del y
        for fl in a.flavours.split(","):
            os.environ.pop("TM_STAGED_KERNEL", None)
            if fl != "default":
                os.environ["TM_STAGED_KERNEL"] = fl
            ex = tm.Exchanger(P, a.strategy, rank=rank, size=k, device=local, nlocal=1, timeout_s=30)
            lay = ex.layout()
            s = torch.cuda.Stream()
            for _ in range(3):
                ex.exchange(x, s)
            s.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for _ in range(a.inner):
                    ex.exchange(x, s)
            g.replay()
            s.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                e0.record(s)
                for _ in range(a.reps):
                    g.replay()
                e1.record(s)
            s.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / (a.reps * a.inner)
            t = torch.tensor([us], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            code, bits = ex.status(s)
            del g
            dist.barrier()
            ex.finalize()
            if rank == 0:
                print(json.dumps({"P": P, "k": k, "procs": k, "strategy": a.strategy, "flavour": fl,
                                  "kernel": NAMES[lay["staged_kernel"]], "L": lay["seg_len"],
                                  "C": lay["ctas_per_rank"], "us_max_over_ranks": float(t.item()),
                                  "nccl_allreduce_us": nccl_us, "fp32_bytes": 4 * P,
                                  "status": code}), flush=True)
        del x
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
