"""Multi-process exchange: one process per rank (nlocal = 1), peers reached through
CUDA IPC mappings, flags in peer memory -- the north-star deployment.  On the
one-GPU test box all processes share cuda:0 (IPC across processes on one device;
the kernels are time-sliced, so this checks correctness, not speed).  With
TM_TEST_MPS=1 and a CUDA MPS daemon running, the processes' kernels run
concurrently instead (real cross-process races on the flags and data)."""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from gpu_helpers import assert_bitwise, fuzz_cases
from oracle import exchange as ox
from paper_1605_08325_b200.inputs import worker_buffer

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def nccl_shared_gpu_env(r, k):
    """NCCL refuses two ranks on one device of one host ("Duplicate GPU detected")
    but identifies a host by NCCL_HOSTID: when the k processes must share fewer
    GPUs, each gets its own host id, so NCCL (AR's ncclAllReduce, the TM_AG_NCCL
    allgather, torch's NCCL process groups) runs with its socket transport over
    loopback.  tools/nccl_one_gpu_probe.py shows it on a one-GPU box."""
    import torch
    if torch.cuda.device_count() >= k:
        return {}
    return {"NCCL_HOSTID": f"tm-test-rank-{r}", "NCCL_SOCKET_IFNAME": "lo", "NCCL_IB_DISABLE": "1"}


def launch(tmp_path, k, strategy, P, dist, mode="normal", timeout=240, extra_env=None):
    port = _free_port()
    procs = []
    extra = dict(extra_env or {})
    if os.environ.get("TM_TEST_MPS") == "1":
        # the processes run concurrently under a CUDA MPS daemon started by the
        # caller: each keeps 1/k of the co-resident CTAs
        extra.setdefault("TM_PROCS_PER_GPU", str(k))
    for r in range(k):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(k), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), LOCAL_RANK=str(r), **nccl_shared_gpu_env(r, k), **extra)
        # TM_TEST_SANITIZER=memcheck|synccheck|racecheck: every worker under
        # compute-sanitizer (its log next to the rank's results)
        san = os.environ.get("TM_TEST_SANITIZER")
        pre = (["compute-sanitizer", "--tool", san, "--error-exitcode", "9",
                "--log-file", os.path.join(str(tmp_path), f"san_{san}_rank{r}.txt")] if san else [])
        procs.append(subprocess.Popen(pre + [sys.executable, os.path.join(HERE, "mp_worker.py"), str(tmp_path),
                                             strategy, str(P), dist, mode], env=env))
    try:
        for p in procs:
            p.wait(timeout=timeout)
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    assert all(p.returncode == 0 for p in procs), [p.returncode for p in procs]
    res = [json.load(open(os.path.join(tmp_path, f"rank{r}.json"))) for r in range(k)]
    return res


KERNEL_ID = {"reg": 0, "tma": 1, "ws": 2, "tmaws": 3, "oneshot": 4, "ll": 5, "ll2": 6}


@pytest.mark.parametrize("strategy,k,op,kernel", [("asa16", 2, "avg", "ws"), ("asa", 2, "avg", "ws"),
                                                  ("asa16", 3, "avg", "ws"), ("asa16", 2, "sum", "ws"),
                                                  ("asa16", 2, "range", "ws"), ("asa16", 2, "avg", "tma"),
                                                  ("asa", 3, "range", "tma"), ("asa16", 2, "avg", "reg"),
                                                  ("asa", 3, "range", "reg"), ("asa16", 2, "avg", "tmaws"),
                                                  ("asa", 3, "range", "tmaws"), ("asa16", 3, "sum", "tmaws"),
                                                  ("asa16", 2, "avg", "oneshot"), ("asa", 3, "range", "oneshot"),
                                                  ("asa16", 4, "sum", "oneshot"), ("asa16", 2, "avg", "ll"),
                                                  ("asa", 3, "range", "ll"), ("asa16", 4, "sum", "ll"),
                                                  ("asa16", 2, "avg", "ll2"), ("asa", 3, "range", "ll2"),
                                                  ("asa16", 4, "sum", "ll2")])
def test_multiprocess_bitwise(tmp_path, strategy, k, op, kernel):
    P = 100_003
    env = {"TM_STAGED_KERNEL": kernel}
    res = launch(tmp_path, k, strategy, P, "D2", mode=("normal" if op == "avg" else op), extra_env=env)
    for r in range(k):
        assert res[r]["layout"]["staged_kernel"] == KERNEL_ID[kernel]
    op = "sum" if op == "sum" else "avg"  # bucketed ranges give the full exchange
    X = [worker_buffer(P, "D2", r, config=50) for r in range(k)]
    want = X
    for _ in range(3):
        want = ox.exchange(want, strategy, op=op)
    for r in range(k):
        assert res[r]["code"] == 0, res[r]
        got = np.load(os.path.join(tmp_path, f"rank{r}.npy"))
        assert_bitwise(got, want[r], f"{strategy} rank {r}")


@pytest.mark.parametrize("strategy,k,mode,kernel", [("asa16", 2, "bsp", "ws"), ("asa16", 3, "bspmom", "ws"),
                                                    ("asa", 2, "bsp", "tma"), ("asa16", 3, "bspmom", "tma"),
                                                    ("asa16", 2, "bsp", "reg"), ("asa", 3, "bspmom", "reg"),
                                                    ("asa16", 3, "bspmom", "tmaws"), ("asa16", 3, "bspmom", "oneshot"),
                                                    ("asa", 2, "bsp", "oneshot"), ("asa16", 3, "bspmom", "ll"),
                                                    ("asa", 2, "bsp", "ll"), ("asa16", 3, "bspmom", "ll2"),
                                                    ("asa", 2, "bsp", "ll2")])
def test_multiprocess_bsp_fused_bitwise(tmp_path, strategy, k, mode, kernel):
    """tm_bsp_step across processes: the momentum-SGD step is fused into the
    staged kernel's pre-cast; two iterations vs oracle/bsp.py."""
    from oracle.bsp import bsp_iteration
    P = 100_003
    env = {"TM_STAGED_KERNEL": kernel}
    res = launch(tmp_path, k, strategy, P, "D2", mode=mode, extra_env=env)
    W = [worker_buffer(P, "D2", r, config=50) for r in range(k)]
    V = [worker_buffer(P, "D4", r, config=52) for r in range(k)]
    G = [worker_buffer(P, "D2", r, config=53) for r in range(k)]
    for _ in range(2):
        W, V = bsp_iteration(W, V, G, 0.01, 0.9, strategy, exchange_momentum=(mode == "bspmom"))
    for r in range(k):
        assert res[r]["code"] == 0, res[r]
        assert res[r]["layout"]["staged_kernel"] == KERNEL_ID[kernel]
        assert_bitwise(np.load(os.path.join(tmp_path, f"rank{r}.npy")), W[r], f"w rank {r}")
        assert_bitwise(np.load(os.path.join(tmp_path, f"vel{r}.npy")), V[r], f"v rank {r}")


@pytest.mark.parametrize("strategy,k,mode,kernel", [("asa16", 2, "normal", "ws"), ("asa", 3, "range", "tma"),
                                                    ("asa16", 3, "bspmom", "reg")])
def test_multiprocess_copy_engine_allgather(tmp_path, strategy, k, mode, kernel):
    """TM_ALLGATHER=ce across processes: the copy engines pull the peers' averaged
    segments through the IPC mappings (the NVLink copy path on a multi-GPU box)."""
    P = 100_003
    env = {"TM_ALLGATHER": "ce", "TM_STAGED_KERNEL": kernel}
    res = launch(tmp_path, k, strategy, P, "D2", mode=mode, extra_env=env)
    for r in range(k):
        assert res[r]["code"] == 0, res[r]
        assert res[r]["layout"]["allgather"] == 1
    if mode.startswith("bsp"):
        from oracle.bsp import bsp_iteration
        W = [worker_buffer(P, "D2", r, config=50) for r in range(k)]
        V = [worker_buffer(P, "D4", r, config=52) for r in range(k)]
        G = [worker_buffer(P, "D2", r, config=53) for r in range(k)]
        for _ in range(2):
            W, V = bsp_iteration(W, V, G, 0.01, 0.9, strategy, exchange_momentum=True)
        want = W
    else:
        want = [worker_buffer(P, "D2", r, config=50) for r in range(k)]
        for _ in range(3):
            want = ox.exchange(want, strategy)
    for r in range(k):
        assert_bitwise(np.load(os.path.join(tmp_path, f"rank{r}.npy")), want[r], f"rank {r}")


@pytest.mark.parametrize("strategy,k,kernel", [("asa16", 2, "tmaws"), ("asa", 3, "reg"), ("asa16", 4, "tma")])
def test_multiprocess_nccl_allgather(tmp_path, strategy, k, kernel):
    """TM_ALLGATHER=nccl: ncclAllGather of the averaged segments, then the widen
    kernel (the north star's NCCL fallback for a6).  On a one-GPU box the ranks'
    NCCL traffic goes over its socket transport (nccl_shared_gpu_env)."""
    P = 100_003
    res = launch(tmp_path, k, strategy, P, "D2", extra_env={"TM_ALLGATHER": "nccl", "TM_STAGED_KERNEL": kernel})
    want = [worker_buffer(P, "D2", r, config=50) for r in range(k)]
    for _ in range(3):
        want = ox.exchange(want, strategy)
    for r in range(k):
        assert res[r]["code"] == 0 and res[r]["layout"]["allgather"] == 2, res[r]
        assert_bitwise(np.load(os.path.join(tmp_path, f"rank{r}.npy")), want[r], f"rank {r}")


@pytest.mark.parametrize("k", [2, 3, 4, 8])
def test_multiprocess_ar_nccl_within_q11(tmp_path, k):
    """AR across processes is NCCL's allreduce (ncclAvg, a8): its summation order
    is NCCL's, so it is checked against the oracle within reading Q11.  On a
    one-GPU box the k processes share cuda:0 and NCCL moves the data over its
    socket transport (nccl_shared_gpu_env); the library's path -- dlopen'ed
    NCCL, the unique id carried in rank 0's bootstrap blob, ncclCommInitRank,
    ncclAllReduce(ncclAvg) on the caller's stream -- is the deployment's."""
    from gpu_helpers import q11_bound
    P = 100_003
    res = launch(tmp_path, k, "ar", P, "D2")
    X = [worker_buffer(P, "D2", r, config=50) for r in range(k)]
    want = X
    bounds = []
    for _ in range(3):
        bounds.append(q11_bound(want))
        want = ox.exchange(want, "ar")
    got = [np.load(os.path.join(tmp_path, f"rank{r}.npy")) for r in range(k)]
    # three exchanges in a row: each one's order error is bounded by Q11 of its own
    # inputs; the errors of earlier exchanges are averaged (not amplified) by later ones
    tol = sum(bounds)
    for r in range(k):
        assert res[r]["code"] == 0, res[r]
        assert res[r]["layout"]["strategy"] == 0
        assert np.all(np.abs(got[r].astype(np.float64) - want[r]) <= tol), f"rank {r}"


@pytest.mark.parametrize("k", [2, 4, 8])
def test_multiprocess_ar_nccl_exact_inputs_bitwise(tmp_path, k):
    """AR == ASA == the exact mean in exact arithmetic (SURVEY 8(c) pin): on
    integers in [-256, 256] every summation order is exact and /k (k a power of
    two) is exact, so NCCL's allreduce must equal the oracle BITWISE whatever
    its order."""
    P = 65_537
    res = launch(tmp_path, k, "ar", P, "D5")
    want = [worker_buffer(P, "D5", r, config=50) for r in range(k)]
    for _ in range(3):
        want = ox.exchange(want, "asa")
    for r in range(k):
        assert res[r]["code"] == 0, res[r]
        assert_bitwise(np.load(os.path.join(tmp_path, f"rank{r}.npy")), want[r], f"rank {r}")


@pytest.mark.parametrize("k,kernel", [(4, "tmaws"), (8, "tmaws"), (8, "reg")])
def test_multiprocess_k4_k8_cross_rank_identity(tmp_path, k, kernel):
    """k = 4 and 8 processes (on a one-GPU box they share cuda:0,
    time-sliced): bitwise parity with the oracle and every rank's buffer
    bitwise identical (cross-rank identity)."""
    P = 60_001 if kernel == "reg" else 300_007
    res = launch(tmp_path, k, "asa16", P, "D2", extra_env={"TM_STAGED_KERNEL": kernel}, timeout=600)
    want = [worker_buffer(P, "D2", r, config=50) for r in range(k)]
    for _ in range(3):
        want = ox.exchange(want, "asa16")
    got = [np.load(os.path.join(tmp_path, f"rank{r}.npy")) for r in range(k)]
    for r in range(k):
        assert res[r]["code"] == 0, res[r]
        assert res[r]["layout"]["staged_kernel"] == KERNEL_ID[kernel]
        assert_bitwise(got[r], want[r], f"rank {r}")
        assert_bitwise(got[r], got[0], f"rank {r} vs rank 0")


@pytest.mark.parametrize("kernel", ["reg", "tma", "ws", "tmaws", "oneshot", "ll", "ll2"])
def test_multiprocess_timeout_instead_of_hang(tmp_path, kernel):
    """Fault injection: rank 1 never calls tm_exchange; rank 0's
    kernel times out in its first barrier, sets TM_E_TIMEOUT and exits -- every
    staged flavour (the warp-specialised ones time out in the reducer group)."""
    P = 4096 if kernel in ("reg", "oneshot", "ll", "ll2") else 300_007
    res = launch(tmp_path, 2, "asa16", P, "D1", mode="skip1", extra_env={"TM_STAGED_KERNEL": kernel})
    assert res[0]["code"] == 7 and res[0]["bits"] & 4  # TM_E_TIMEOUT


def test_multiprocess_mismatch_detected(tmp_path):
    """Ranks disagreeing on nparams fail the bootstrap with TM_E_MISMATCH."""
    res = launch(tmp_path, 2, "asa", 4096, "D1", mode="mismatch")
    assert any(r.get("init_error") == 6 for r in res), res


@pytest.mark.parametrize("mode", ["concurrent", "concurrent_exact"])
@pytest.mark.parametrize("k", [2, 4])
def test_multiprocess_concurrent_easgd_admissible(tmp_path, mode, k):
    """k processes update the sharded centre at once (system-scope atomic adds
    into the peers' shards over the IPC mappings, reading Q15):
    every element of every worker and of the centre is bitwise one of the
    oracle's interleavings (oracle.easgd.easgd_concurrent_admissible; the fast
    mode against the flushing add, the exact mode against the IEEE add)."""
    from oracle.easgd import easgd_concurrent_admissible
    P = 100_003
    res = launch(tmp_path, k, "easgd", P, "D1", mode=mode)
    W = [worker_buffer(P, "D1", r, config=51) for r in range(k)]
    c0 = worker_buffer(P, "D1", 99, config=51)
    L = res[0]["seg_len"]
    gW = [np.load(os.path.join(tmp_path, f"rank{r}.npy")) for r in range(k)]
    gc = np.concatenate([np.load(os.path.join(tmp_path, f"shard{r}.npy")) for r in range(k)])[:P]
    assert L * (k - 1) < P
    ok = easgd_concurrent_admissible(W, c0, np.float32(0.3), gW, gc,
                                     add="ftz" if mode == "concurrent" else "ieee")
    assert ok.all(), f"{int((~ok).sum())} of {P} elements are no interleaving's result"


def test_multiprocess_sharded_easgd(tmp_path):
    """EASGD centre sharded across two processes; worker updates reach the peer's
    shard through the IPC mapping; bitwise the oracle's serial order."""
    from oracle.easgd import easgd_sequence
    P, k = 100_003, 2
    res = launch(tmp_path, k, "easgd", P, "D1")
    W = [worker_buffer(P, "D1", r, config=51) for r in range(k)]
    c0 = worker_buffer(P, "D1", 99, config=51)
    wW, wc = easgd_sequence(W, c0, 0.3, [0, 1])
    L = res[0]["seg_len"]
    for r in range(k):
        assert_bitwise(np.load(os.path.join(tmp_path, f"rank{r}.npy")), wW[r], f"worker {r}")
        sh = np.load(os.path.join(tmp_path, f"shard{r}.npy"))
        assert_bitwise(sh, wc[r * L: r * L + sh.shape[0]], f"shard {r}")


def test_multiprocess_locked_easgd(tmp_path):
    """Two processes update the sharded centre at the same time with per-chunk
    locks over IPC (system-scope atomics); each process logs its own arrival
    positions; the merged order reproduces every chunk bitwise."""
    from oracle.easgd import easgd_sequence
    P, k = 300_007, 2
    res = launch(tmp_path, k, "easgd", P, "D1", mode="locked")
    W = [worker_buffer(P, "D1", r, config=51) for r in range(k)]
    c0 = worker_buffer(P, "D1", 99, config=51)
    L = res[0]["seg_len"]
    nch = -(-L // 4096)
    logs = [np.load(os.path.join(tmp_path, f"log{r}.npy")) for r in range(k)]
    merged = np.maximum(logs[0], logs[1])
    gW = [np.load(os.path.join(tmp_path, f"rank{r}.npy")) for r in range(k)]
    shards = [np.load(os.path.join(tmp_path, f"shard{r}.npy")) for r in range(k)]
    gc = np.concatenate(shards)[:P]
    for s in range(k):
        for q in range(nch):
            lo, hi = s * L + q * 4096, min(s * L + min(L, (q + 1) * 4096), P)
            if lo >= hi:
                continue
            order = [int(v) for v in merged[(s * nch + q) * k:(s * nch + q + 1) * k]]
            assert sorted(order) == [0, 1], order
            ws, cc = easgd_sequence([w[lo:hi] for w in W], c0[lo:hi], 0.3, order)
            assert_bitwise(gc[lo:hi], cc, f"chunk ({s},{q})")
            for r in range(k):
                assert_bitwise(gW[r][lo:hi], ws[r])


@pytest.mark.parametrize("k", [2, 3])
def test_multiprocess_async_easgd_loop(tmp_path, k):
    """The asynchronous EASGD loop: every process runs rounds of
    tau local SGD steps and a per-worker atomic elastic exchange with the sharded
    centre, with random delays; replaying every chunk's logged arrival order in
    oracle.easgd.easgd_async_replay reproduces workers and centre bitwise."""
    import mp_worker as mw
    from oracle.easgd import easgd_async_replay
    P = 150_001
    res = launch(tmp_path, k, "easgd", P, "D1", mode="async")
    W = [worker_buffer(P, "D1", r, config=51) for r in range(k)]
    T = [worker_buffer(P, "D1", 10 + r, config=54) for r in range(k)]
    c0 = worker_buffer(P, "D1", 99, config=51)
    L = res[0]["seg_len"]
    nch = -(-L // 4096)
    per = mw.ASYNC_ROUNDS * k
    merged = np.max(np.stack([np.load(os.path.join(tmp_path, f"log{r}.npy")) for r in range(k)]), axis=0)
    gW = [np.load(os.path.join(tmp_path, f"rank{r}.npy")) for r in range(k)]
    gc = np.concatenate([np.load(os.path.join(tmp_path, f"shard{r}.npy")) for r in range(k)])[:P]
    orders_seen = set()
    for s_ in range(k):
        for q in range(nch):
            lo, hi = s_ * L + q * 4096, min(s_ * L + min(L, (q + 1) * 4096), P)
            if lo >= hi:
                continue
            order = [int(v) for v in merged[(s_ * nch + q) * per:(s_ * nch + q + 1) * per]]
            assert sorted(order) == sorted(list(range(k)) * mw.ASYNC_ROUNDS), order
            orders_seen.add(tuple(order))
            ws, cc = easgd_async_replay([w[lo:hi] for w in W], c0[lo:hi], [t[lo:hi] for t in T],
                                        mw.ASYNC_ETA, mw.ASYNC_TAU, 0.5 / k, order)
            assert_bitwise(gc[lo:hi], cc, f"centre chunk ({s_},{q})")
            for r in range(k):
                assert_bitwise(gW[r][lo:hi], ws[r], f"worker {r} chunk ({s_},{q})")
    assert len(orders_seen) >= 1


@pytest.mark.parametrize("strategy,kernel", [("asa16", "ws"), ("asa", "reg"), ("asa16", "tma"),
                                             ("asa16", "tmaws"), ("asa16", "oneshot"), ("asa16", "ll"),
                                             ("asa", "ll2")])
def test_multiprocess_stress_random_delays(tmp_path, strategy, kernel):
    """STRESS_ITERS (60; TM_STRESS_ITERS overrides) back-to-back exchanges per rank, each after a per-rank delta and a random
    host delay on half of them: every rank ends bitwise at the oracle's sequence."""
    from mp_worker import STRESS_ITERS
    P, k = 50_003, 2
    env = {"TM_STAGED_KERNEL": kernel}
    res = launch(tmp_path, k, strategy, P, "D2", mode="stress", extra_env=env, timeout=600)
    X = [worker_buffer(P, "D2", r, config=50) for r in range(k)]
    for it in range(STRESS_ITERS):
        X = [np.add(X[r], np.random.default_rng([1605, r, it]).standard_normal(P).astype(np.float32)
                    * np.float32(1e-3), dtype=np.float32) for r in range(k)]
        X = ox.exchange(X, strategy)
    for r in range(k):
        assert res[r]["code"] == 0, res[r]
        assert_bitwise(np.load(os.path.join(tmp_path, f"rank{r}.npy")), X[r], f"rank {r}")


@pytest.mark.parametrize("strategy,k,kernel", [("asa16", 2, "tmaws"), ("asa", 3, "tma"), ("asa16", 4, "oneshot"),
                                               ("asa16", 3, "ll"), ("asa16", 4, "ll2")])
def test_multiprocess_bootstrap_selfcheck(tmp_path, strategy, k, kernel):
    """The bootstrap's known-answer probe passes on every rank (tm_layout
    selfcheck = 1) and the chosen flavour stays."""
    P = 100_003
    res = launch(tmp_path, k, strategy, P, "D2", extra_env={"TM_STAGED_KERNEL": kernel})
    want = [worker_buffer(P, "D2", r, config=50) for r in range(k)]
    for _ in range(3):
        want = ox.exchange(want, strategy)
    for r in range(k):
        assert res[r]["code"] == 0, res[r]
        assert res[r]["layout"]["selfcheck"] == 1 and res[r]["layout"]["staged_kernel"] == KERNEL_ID[kernel]
        assert_bitwise(np.load(os.path.join(tmp_path, f"rank{r}.npy")), want[r], f"rank {r}")


@pytest.mark.parametrize("strategy,k,kernel,bad,P", [("asa16", 2, "tmaws", 1, 100_003), ("asa", 3, "tma", 0, 100_003),
                                                     ("asa16", 4, "oneshot", 3, 100_003),
                                                     ("asa16", 6, "ll", 2, 600_001)])
def test_multiprocess_selfcheck_fault_falls_back(tmp_path, strategy, k, kernel, bad, P):
    """Fault injection (TM_SELFCHECK_FAULT=r: rank r reports a probe mismatch):
    the vote through peer memory reaches every rank, ALL ranks fall back to the
    register flavour together (selfcheck = 2, staged_kernel = 0), the re-run
    probe passes, and the exchanges that follow are bitwise the oracle's.  The
    k = 6 LL case has more CTAs per rank (587) than the register kernel keeps
    co-resident at k = 6 (3 per SM): the fallback shrinks C with it."""
    res = launch(tmp_path, k, strategy, P, "D2",
                 extra_env={"TM_STAGED_KERNEL": kernel, "TM_SELFCHECK_FAULT": str(bad)})
    want = [worker_buffer(P, "D2", r, config=50) for r in range(k)]
    for _ in range(3):
        want = ox.exchange(want, strategy)
    for r in range(k):
        assert res[r]["code"] == 0, res[r]
        assert res[r]["layout"]["selfcheck"] == 2 and res[r]["layout"]["staged_kernel"] == 0, res[r]
        assert_bitwise(np.load(os.path.join(tmp_path, f"rank{r}.npy")), want[r], f"rank {r}")


def test_multiprocess_allgather_decision_table(tmp_path):
    """TM_AG_TABLE (the allgather decision step): without TM_ALLGATHER every rank
    takes the mode of the first matching "k L_max mode" rule -- here the copy
    engines for k = 2 -- and the exchange stays bitwise."""
    table = tmp_path / "ag_table.txt"
    table.write_text("# k L_max mode\n4 1000000000 nccl\n2 100 sm\n2 1000000000 ce\n")
    P, k = 100_003, 2
    res = launch(tmp_path, k, "asa16", P, "D2", extra_env={"TM_AG_TABLE": str(table), "TM_STAGED_KERNEL": "tma"})
    want = [worker_buffer(P, "D2", r, config=50) for r in range(k)]
    for _ in range(3):
        want = ox.exchange(want, "asa16")
    for r in range(k):
        assert res[r]["code"] == 0 and res[r]["layout"]["allgather"] == 1, res[r]
        assert_bitwise(np.load(os.path.join(tmp_path, f"rank{r}.npy")), want[r], f"rank {r}")


@pytest.mark.parametrize("strategy,k,kernel", [("asa16", 2, "oneshot"), ("asa16", 3, "tmaws"), ("asa", 4, "oneshot"),
                                               ("asa16", 2, "reg"), ("asa", 3, "ll"), ("asa16", 3, "ll2")])
def test_multiprocess_cuda_graph_replays(tmp_path, strategy, k, kernel):
    """Each process captures 4 x (its delta, exchange) in a CUDA graph and
    replays it 3 times: device-side epochs (and the one-shot kernel's device call
    parity) keep the replayed exchanges collective; every rank ends bitwise at
    the oracle's sequence of 13 exchanges."""
    import mp_worker as mw
    P = 40_003
    res = launch(tmp_path, k, strategy, P, "D2", mode="graph", extra_env={"TM_STAGED_KERNEL": kernel})
    X = [worker_buffer(P, "D2", r, config=50) for r in range(k)]
    D = [np.random.default_rng([1606, r]).standard_normal(P).astype(np.float32) * np.float32(1e-3)
         for r in range(k)]
    X = ox.exchange(X, strategy)
    for _ in range(mw.GRAPH_REPLAYS):
        for j in range(mw.GRAPH_PER):
            X = [(np.subtract if j % 2 else np.add)(X[r], D[r], dtype=np.float32) for r in range(k)]
            X = ox.exchange(X, strategy)
    for r in range(k):
        assert res[r]["code"] == 0, res[r]
        assert res[r]["layout"]["staged_kernel"] == KERNEL_ID[kernel]
        assert_bitwise(np.load(os.path.join(tmp_path, f"rank{r}.npy")), X[r], f"rank {r}")


@pytest.mark.parametrize("k", [2, 3, 4, 5, 8])
def test_multiprocess_fuzz_bitwise(tmp_path, k):
    """k processes (one rank each), seeded random combinations of size, strategy,
    op, flavour, distribution, buckets and CTA budgets (or two BSP iterations),
    each case on a fresh exchanger (bootstrap and self-check included), bitwise vs
    the oracle on every rank."""
    pmax = 1 << 18
    res = launch(tmp_path, k, "asa16", pmax, "D1", mode="fuzz", timeout=600)
    from oracle.bsp import bsp_iteration
    for i, c in enumerate(fuzz_cases(k, pmax)):
        if c["bsp"]:
            b = c["bsp"]
            W = [worker_buffer(c["P"], c["dist"], r, config=800 + 4 * i) for r in range(k)]
            V = [worker_buffer(c["P"], "D4", r, config=801 + 4 * i) for r in range(k)]
            G = [worker_buffer(c["P"], "D2", r, config=802 + 4 * i) for r in range(k)]
            for _ in range(2):
                W, V = bsp_iteration(W, V, G, np.float32(b["lr"]), np.float32(b["mu"]), c["strategy"],
                                     exchange_momentum=b["mom"])
            for r in range(k):
                assert res[r][f"code{i}_0"] == 0, (i, c, res[r])
                assert res[r][f"selfcheck{i}"] == 1, (i, c, res[r])
                for name, want in (("w", W[r]), ("v", V[r])):
                    got = np.load(os.path.join(tmp_path, f"fuzz{i}_{name}_rank{r}.npy"))
                    assert_bitwise(got, want, f"mp fuzz bsp k={k} case {i} {c} {name} rank {r}")
            continue
        for n, (off, cnt, _) in enumerate(c["calls"]):
            X = [worker_buffer(c["P"], c["dist"], r, config=800 + 4 * i + n) for r in range(k)]
            want = [x.copy() for x in X]
            if cnt:
                seg = ox.exchange([x[off:off + cnt] for x in X], c["strategy"], op=c["op"])
                for r in range(k):
                    want[r][off:off + cnt] = seg[r]
            for r in range(k):
                assert res[r][f"code{i}_{n}"] == 0, (i, n, c, res[r])
                assert res[r][f"selfcheck{i}"] == 1, (i, c, res[r])  # the flavour's probe passed
                if c["flavour"]:
                    assert res[r][f"kernel{i}"] == KERNEL_ID[c["flavour"]], (i, c, res[r])
                got = np.load(os.path.join(tmp_path, f"fuzz{i}_{n}_rank{r}.npy"))
                assert_bitwise(got, want[r], f"mp fuzz k={k} case {i} {c} call {n} rank {r}")
