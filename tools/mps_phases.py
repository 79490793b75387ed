#!/usr/bin/env python
"""Phase stamps of one staged exchange with k processes running concurrently on
one GPU under CUDA MPS (launched by torchrun; gloo for the bootstrap).  Rank 0
prints the medians over all ranks' CTAs, like tools/phases.py.

    TM_PROCS_PER_GPU=8 TM_STAGED_KERNEL=tmaws torchrun --nproc-per-node 8 tools/mps_phases.py
"""

import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1605_08325_b200 import tm  # noqa: E402

NAMES = ["start", "cast", "ready", "reduce", "reduced", "end"]


def main():
    rank, k = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo")
    torch.cuda.set_device(0)
    P = int(os.environ.get("TM_PHASES_P", "60965224"))
    x = torch.randn(P, device="cuda") * 0.01
    ex = tm.Exchanger(P, "asa16", rank=rank, size=k, device=0, nlocal=1)
    C = ex.layout()["ctas_per_rank"]
    log = torch.zeros(C * 8, dtype=torch.int64, device="cuda")
    for _ in range(5):
        ex.exchange(x)
    torch.cuda.synchronize()
    dist.barrier()
    tm.tm_set_phase_log(log)
    ex.exchange(x)
    torch.cuda.synchronize()
    tm.tm_set_phase_log(None)
    st = log.cpu().numpy().reshape(C, 8)[:, :6]
    allst = [None] * k
    dist.all_gather_object(allst, st)
    if rank == 0:
        st = np.concatenate(allst).astype(np.int64)
        t0 = st[:, 0].min()
        res = {"kernel": ["reg", "tma", "ws", "tmaws"][ex.layout()["staged_kernel"]], "processes": k,
               "ctas": int(st.shape[0]), "span_us": round((st[:, 5].max() - t0) / 1e3, 1),
               "start_spread_us": round((st[:, 0].max() - t0) / 1e3, 1)}
        for i in range(1, 6):
            if st[:, i].max() == 0:
                continue
            prev = i - 1
            while st[:, prev].max() == 0:
                prev -= 1
            d = (st[:, i] - st[:, prev]) / 1e3
            res[f"{NAMES[prev]}->{NAMES[i]}_us_median"] = round(float(np.median(d)), 1)
            res[f"{NAMES[prev]}->{NAMES[i]}_us_max"] = round(float(d.max()), 1)
        print(json.dumps(res), flush=True)
    dist.barrier()
    ex.finalize()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
