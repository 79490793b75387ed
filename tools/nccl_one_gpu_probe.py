#!/usr/bin/env python
"""Probe: can NCCL run k ranks whose processes share ONE GPU?  NCCL refuses two
ranks on one device of one host ("Duplicate GPU detected"), but it identifies a
host by NCCL_HOSTID when set, so giving every process its own host id makes the
ranks look like separate hosts and NCCL moves the data over its socket
transport (loopback).  Used by the tests to exercise the cross-process NCCL
paths (AR ncclAllReduce/ncclAvg, the TM_AG_NCCL allgather) on a one-GPU box.

    python tools/nccl_one_gpu_probe.py [k]
"""
import os
import socket
import subprocess
import sys

import torch


def child():
    import torch.distributed as dist
    r, k = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    x = torch.full((1 << 20,), float(r + 1), device="cuda")
    dist.all_reduce(x)
    torch.cuda.synchronize()
    ok = bool((x == k * (k + 1) / 2).all())
    print(f"rank {r}: allreduce ok={ok}", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


def main():
    if os.environ.get("PROBE_CHILD"):
        return child()
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ps = []
    for r in range(k):
        env = dict(os.environ, PROBE_CHILD="1", RANK=str(r), WORLD_SIZE=str(k), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), NCCL_HOSTID=f"tm-rank-{r}", NCCL_SOCKET_IFNAME="lo",
                   NCCL_IB_DISABLE="1")
        ps.append(subprocess.Popen([sys.executable, __file__], env=env))
    rc = [p.wait(timeout=300) for p in ps]
    print("rc", rc)
    sys.exit(max(rc))


if __name__ == "__main__":
    main()
