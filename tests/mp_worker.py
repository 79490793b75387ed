"""One rank of a multi-process exchange (one process per rank, nlocal = 1),
bootstrapped over a gloo process group: CUDA IPC handles are swapped with
all_gather_object.  Used by tests/test_gpu_multiprocess.py; on a one-GPU box
every rank uses cuda:0 (IPC between processes on one device), on a multi-GPU
box rank r uses cuda:r.

argv: outdir strategy P dist mode      (mode: normal | sum | range | locked | concurrent | concurrent_exact | async | skip1 | mismatch | stress | bsp | bspmom | graph | fuzz)
"""

import json
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1605_08325_b200 import tm  # noqa: E402
from paper_1605_08325_b200.inputs import worker_buffer  # noqa: E402

STRESS_ITERS = int(os.environ.get("TM_STRESS_ITERS", "60"))
ASYNC_ROUNDS, ASYNC_TAU, ASYNC_ETA = 6, 2, 0.25
GRAPH_PER, GRAPH_REPLAYS = 4, 3


def main():
    outdir, strategy, P, dist_name, mode = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4], sys.argv[5]
    rank = int(os.environ["RANK"])
    size = int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo", rank=rank, world_size=size)
    ndev = torch.cuda.device_count()
    device = rank % ndev
    torch.cuda.set_device(device)
    result = {"rank": rank, "device": device}
    Pr = P + (1 if (mode == "mismatch" and rank == 1) else 0)
    try:
        ex = tm.Exchanger(Pr, strategy, rank=rank, size=size, device=device, nlocal=1,
                          timeout_s=(1.0 if mode == "skip1" else 20.0),
                          op=("sum" if mode == "sum" else "avg"))
    except tm.TmError as e:
        result["init_error"] = e.code
        json.dump(result, open(os.path.join(outdir, f"rank{rank}.json"), "w"))
        dist.barrier()
        return
    if strategy == "easgd":
        # sharded centre across processes: each rank fills its own shard, then the
        # workers update the whole centre one at a time (rank order), remote
        # shards through the IPC mapping.
        c0 = worker_buffer(P, dist_name, 99, config=51)
        L = ex.layout()["seg_len"]
        mine = ex.center_shard(rank)
        mine.copy_(torch.from_numpy(c0[rank * L: rank * L + mine.numel()]))
        x = torch.from_numpy(worker_buffer(P, dist_name, rank, config=51)).cuda()
        torch.cuda.synchronize()
        log = None
        if mode == "async":
            # The asynchronous EASGD loop: ROUNDS
            # rounds of TAU local SGD steps on the synthetic quadratic objective
            # |x - t_r|^2 / 2 (torch ops, one rounding each), then a per-worker
            # atomic elastic exchange with the sharded centre in arrival order;
            # random host delays vary the arrival order between chunks and rounds.
            import random
            rnd = random.Random(77 + rank)
            t = torch.from_numpy(worker_buffer(P, dist_name, 10 + rank, config=54)).cuda()
            nch = -(-L // 4096)
            log = torch.full((size * nch * ASYNC_ROUNDS * size,), -1, dtype=torch.int32, device="cuda")
            tm.tm_easgd_set_order_log(log, ASYNC_ROUNDS * size)
            dist.barrier()
            for _ in range(ASYNC_ROUNDS):
                for _ in range(ASYNC_TAU):
                    d = x.sub(t)
                    x.sub_(d.mul(ASYNC_ETA))
                if rnd.random() < 0.5:
                    torch.cuda.synchronize()
                    time.sleep(rnd.random() * 0.002)
                tm.tm_easgd_update_locked(x, rank, 0.5 / size)
            torch.cuda.synchronize()
        elif mode in ("concurrent", "concurrent_exact"):  # all workers at once, atomic centre adds
            dist.barrier()
            tm.tm_easgd_update_sharded(x, 0.3, concurrent=(True if mode == "concurrent" else "exact"))
            torch.cuda.synchronize()
        elif mode == "locked":  # all workers at once; per-chunk locks order them
            nch = -(-L // 4096)
            log = torch.full((size * nch * size,), -1, dtype=torch.int32, device="cuda")
            tm.tm_easgd_set_order_log(log, size)
            dist.barrier()
            tm.tm_easgd_update_locked(x, rank, 0.3)
            torch.cuda.synchronize()
        else:
            for w in range(size):
                dist.barrier()
                if w == rank:
                    tm.tm_easgd_update_sharded(x, 0.3)
                    torch.cuda.synchronize()
        dist.barrier()
        if log is not None:
            np.save(os.path.join(outdir, f"log{rank}.npy"), log.cpu().numpy())
        shard = ex.center_shard(rank).cpu().numpy()
        np.save(os.path.join(outdir, f"rank{rank}.npy"), x.cpu().numpy())
        np.save(os.path.join(outdir, f"shard{rank}.npy"), shard)
        result.update({"code": 0, "bits": 0, "seg_len": L})
        json.dump(result, open(os.path.join(outdir, f"rank{rank}.json"), "w"))
        dist.barrier()
        ex.finalize()
        dist.destroy_process_group()
        return
    x = torch.from_numpy(worker_buffer(P, dist_name, rank, config=50)).cuda()
    if mode == "fuzz":
        # seeded random cases (tests/gpu_helpers.py::fuzz_cases), each on
        # an exchanger of its own: init + bootstrap (with the self-check), 1-3
        # calls (full or a bucket with a CTA budget) on fresh inputs, finalize
        ex.finalize()
        from gpu_helpers import fuzz_cases
        for i, c in enumerate(fuzz_cases(size, P)):
            if c["flavour"]:
                os.environ["TM_STAGED_KERNEL"] = c["flavour"]
            else:
                os.environ.pop("TM_STAGED_KERNEL", None)
            ex = tm.Exchanger(c["P"], c["strategy"], rank=rank, size=size, device=device, nlocal=1,
                              timeout_s=20.0, op=c["op"])
            if c["bsp"]:
                b = c["bsp"]
                w = torch.from_numpy(worker_buffer(c["P"], c["dist"], rank, config=800 + 4 * i)).cuda()
                v = torch.from_numpy(worker_buffer(c["P"], "D4", rank, config=801 + 4 * i)).cuda()
                gr = torch.from_numpy(worker_buffer(c["P"], "D2", rank, config=802 + 4 * i)).cuda()
                for _ in range(2):
                    ex.bsp_step(w, v, gr, b["lr"], b["mu"], exchange_momentum=b["mom"])
                code, bits = ex.status()
                result[f"code{i}_0"] = code
                np.save(os.path.join(outdir, f"fuzz{i}_w_rank{rank}.npy"), w.cpu().numpy())
                np.save(os.path.join(outdir, f"fuzz{i}_v_rank{rank}.npy"), v.cpu().numpy())
            for n, (off, cnt, budget) in enumerate([] if c["bsp"] else c["calls"]):
                xi = torch.from_numpy(worker_buffer(c["P"], c["dist"], rank, config=800 + 4 * i + n)).cuda()
                tm.tm_set_range_ctas(budget)
                if off == 0 and cnt == c["P"]:
                    ex.exchange(xi)
                else:
                    ex.exchange_range(xi, off, cnt)
                code, bits = ex.status()
                result[f"code{i}_{n}"] = code
                np.save(os.path.join(outdir, f"fuzz{i}_{n}_rank{rank}.npy"), xi.cpu().numpy())
            lay = ex.layout()
            result[f"kernel{i}"] = lay["staged_kernel"]
            result[f"selfcheck{i}"] = lay["selfcheck"]
            dist.barrier()  # every rank done with the peers' slabs
            ex.finalize()
        result["code"] = 0
        json.dump(result, open(os.path.join(outdir, f"rank{rank}.json"), "w"))
        dist.barrier()
        dist.destroy_process_group()
        return
    if mode in ("bsp", "bspmom"):
        # two BSP iterations (momentum SGD fused into the staged pre-cast, then
        # the exchange of w, and of v for bspmom)
        v = torch.from_numpy(worker_buffer(P, "D4", rank, config=52)).cuda()
        g = torch.from_numpy(worker_buffer(P, dist_name, rank, config=53)).cuda()
        for _ in range(2):
            ex.bsp_step(x, v, g, 0.01, 0.9, exchange_momentum=(mode == "bspmom"))
        code, bits = ex.status()
        result.update({"code": code, "bits": bits, "layout": ex.layout()})
        np.save(os.path.join(outdir, f"rank{rank}.npy"), x.cpu().numpy())
        np.save(os.path.join(outdir, f"vel{rank}.npy"), v.cpu().numpy())
        json.dump(result, open(os.path.join(outdir, f"rank{rank}.json"), "w"))
        dist.barrier()
        ex.finalize()
        dist.destroy_process_group()
        return
    if mode == "graph":
        # GRAPH_PER x (per-rank delta of alternating sign; exchange) captured once in a
        # CUDA graph and replayed GRAPH_REPLAYS times: the epochs and the one-shot
        # kernel's call parity live on the device, so replays stay collective
        d = torch.from_numpy(np.random.default_rng([1606, rank]).standard_normal(P).astype(np.float32)
                             * np.float32(1e-3)).cuda()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            ex.exchange(x, s)  # one eager exchange first (warm-up, and bootstrapped state)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for j in range(GRAPH_PER):
                    x.sub_(d) if j % 2 else x.add_(d)
                    ex.exchange(x, s)
        torch.cuda.current_stream().wait_stream(s)
        for _ in range(GRAPH_REPLAYS):
            dist.barrier()
            g.replay()
        torch.cuda.synchronize()
        code, bits = ex.status()
        result.update({"code": code, "bits": bits, "layout": ex.layout()})
        np.save(os.path.join(outdir, f"rank{rank}.npy"), x.cpu().numpy())
        json.dump(result, open(os.path.join(outdir, f"rank{rank}.json"), "w"))
        dist.barrier()
        del g
        ex.finalize()
        dist.destroy_process_group()
        return
    if mode == "stress":
        # back-to-back exchanges with random host delays between calls on each
        # rank (exercises the epoch / reuse protocol); each iteration
        # first adds a deterministic per-rank delta
        import random
        rnd = random.Random(1000 + rank)
        for it in range(STRESS_ITERS):
            d = np.random.default_rng([1605, rank, it]).standard_normal(P).astype(np.float32) * np.float32(1e-3)
            x.add_(torch.from_numpy(d).cuda())
            if rnd.random() < 0.5:
                torch.cuda.synchronize()
                time.sleep(rnd.random() * 0.003)
            ex.exchange(x)
        code, bits = ex.status()
        result.update({"code": code, "bits": bits, "layout": ex.layout()})
        np.save(os.path.join(outdir, f"rank{rank}.npy"), x.cpu().numpy())
        json.dump(result, open(os.path.join(outdir, f"rank{rank}.json"), "w"))
        dist.barrier()
        ex.finalize()
        dist.destroy_process_group()
        return
    reps = 3
    if mode == "skip1" and rank == 1:
        reps = 0  # never arrives: rank 0 must time out, not hang
    for _ in range(reps):
        if mode == "range":  # three buckets, last first (backward order)
            b1, b2 = P // 3 // 4 * 4, 2 * P // 3 // 4 * 4
            ex.exchange_range(x, b2, P - b2)
            ex.exchange_range(x, b1, b2 - b1)
            ex.exchange_range(x, 0, b1)
        else:
            ex.exchange(x)
        # re-run on fresh inputs so each call is checked
        if _ < reps - 1:
            torch.cuda.synchronize()
    code, bits = ex.status()
    result.update({"code": code, "bits": bits, "layout": ex.layout()})
    np.save(os.path.join(outdir, f"rank{rank}.npy"), x.cpu().numpy())
    json.dump(result, open(os.path.join(outdir, f"rank{rank}.json"), "w"))
    dist.barrier()  # keep every slab alive until all ranks are done
    ex.finalize()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
