"""Seeded random sweep over the exchange's configuration space, bitwise against
the oracle (`-m gpu`).

The other GPU tests walk one axis at a time (sizes, distributions, flavours,
ranges, sum mode, BSP); this one draws COMBINATIONS of them, so an interaction
no axis-wise test reaches (say the one-shot kernel on a budgeted range in sum
mode with specials at k = 7) still meets the oracle.  Every case is fixed by
the seed, so a failure names a reproducible case.

Per case: k in 2..8; P log-uniform in [1, 2^20] (ragged: any residue mod 4 and
mod 256); strategy AR / ASA / ASA16; op avg (AWAGD) or sum (SUBGD, ASA and
ASA16); path direct or staged with any of the five staged flavours (or the
runtime's own choice); distribution D1-D6; then 1-3 calls, each a full
exchange or a bucket [offset, offset + count) with an optional CTA budget,
on fresh inputs, on the default stream or a fresh non-blocking one, each
compared bitwise with oracle/exchange.py on exactly the elements it covers (the
rest must be untouched).  PAPER L237-269 (ASA,
ASA16), L233-237 (AR; a single-process group sums in ascending rank order, so
bitwise too), L384-389 (SUBGD sum).
"""

import os

import numpy as np
import pytest
import torch

from gpu_helpers import assert_bitwise, to_dev, to_host
from oracle import exchange as ox
from oracle.bsp import bsp_iteration
from paper_1605_08325_b200 import tm
from paper_1605_08325_b200.inputs import DISTS, worker_buffers

pytestmark = pytest.mark.gpu

FLAVOURS = [None, "reg", "tma", "ws", "tmaws", "oneshot", "ll", "ll2"]
NCASES = int(os.environ.get("TM_FUZZ_CASES", "384"))
NBSP = int(os.environ.get("TM_FUZZ_BSP_CASES", "64"))


def draw_case(i):
    g = np.random.default_rng([1605, 8325, 777, i])
    k = int(g.integers(2, 9))
    P = int(np.exp(g.uniform(0.0, np.log(1 << 20)))) + int(g.integers(0, 4))
    P = max(1, min(P, 1 << 20))
    strategy = str(g.choice(["ar", "asa", "asa16"], p=[0.2, 0.4, 0.4]))
    op = "sum" if strategy != "ar" and g.random() < 0.3 else "avg"
    path = "direct" if strategy == "ar" or g.random() < 0.3 else "staged"
    flavour = FLAVOURS[int(g.integers(0, len(FLAVOURS)))] if path == "staged" else None
    dist = DISTS[int(g.integers(0, len(DISTS)))]
    calls = []
    for _ in range(int(g.integers(1, 4))):
        if P >= 8 and g.random() < 0.5:
            off = int(g.integers(0, P // 4)) * 4
            cnt = int(g.integers(0, P - off + 1))
            budget = [0, 1, 3, 16][int(g.integers(0, 4))]
            calls.append((off, cnt, budget))
        else:
            calls.append((0, P, 0))
    side = bool(g.random() < 0.5)  # calls on a fresh non-blocking stream
    return dict(k=k, P=P, strategy=strategy, op=op, path=path, flavour=flavour, dist=dist, calls=calls,
                side=side)


@pytest.mark.parametrize("i", range(NCASES))
def test_fuzz_case_bitwise(monkeypatch, i):
    c = draw_case(i)
    k, P, strategy, op = c["k"], c["P"], c["strategy"], c["op"]
    if c["flavour"]:
        monkeypatch.setenv("TM_STAGED_KERNEL", c["flavour"])
    else:
        monkeypatch.delenv("TM_STAGED_KERNEL", raising=False)
    what = f"case {i}: {c}"
    with tm.Exchanger(P, strategy, size=k, nlocal=k, path=c["path"], op=op) as ex:
        for n, (off, cnt, budget) in enumerate(c["calls"]):
            X = worker_buffers(P, k, c["dist"], config=700 + n)
            if op == "sum" and strategy == "asa16":
                # keep the sum inside binary16's range (the overflow status is
                # tested elsewhere); D6's 65504s would overflow a sum of k terms
                X = [np.clip(x, -60000.0 / k, 60000.0 / k).astype(np.float32) for x in X]
            bufs = to_dev(X)
            tm.tm_set_range_ctas(budget)
            st = torch.cuda.Stream() if c["side"] else torch.cuda.current_stream()
            st.wait_stream(torch.cuda.current_stream())
            if off == 0 and cnt == P:
                ex.exchange(bufs, st)
            else:
                ex.exchange_range(bufs, off, cnt, st)
            code, bits = ex.status(st)
            assert code in (tm.TM_OK, tm.TM_E_NONFINITE, tm.TM_E_OVERFLOW16), (what, code, bits)
            got = to_host(bufs)
            want = [x.copy() for x in X]
            if cnt:
                seg = ox.exchange([x[off:off + cnt] for x in X], strategy, op)
                for r in range(k):
                    want[r][off:off + cnt] = seg[r]
            for r in range(k):
                assert_bitwise(got[r], want[r], f"{what} call {n} rank {r}")


@pytest.mark.parametrize("i", range(NBSP))
def test_fuzz_bsp_bitwise(monkeypatch, i):
    """The BSP iteration (momentum-SGD step + exchange)
    on random combinations of k, P, strategy, path / flavour, momentum exchange,
    lr and mu, two iterations (state carries over), bitwise against
    oracle/bsp.py."""
    g = np.random.default_rng([1605, 8325, 778, i])
    k = int(g.integers(2, 9))
    P = max(1, int(np.exp(g.uniform(0.0, np.log(1 << 19)))) + int(g.integers(0, 4)))
    strategy = str(g.choice(["ar", "asa", "asa16"], p=[0.2, 0.4, 0.4]))
    path = "direct" if strategy == "ar" or g.random() < 0.4 else "staged"
    flavour = FLAVOURS[int(g.integers(0, len(FLAVOURS)))] if path == "staged" else None
    mom = bool(g.random() < 0.5)
    lr = float(np.float32(g.choice([0.01, 0.05, 0.3])))
    mu = float(np.float32(g.choice([0.0, 0.9, 0.99])))
    if flavour:
        monkeypatch.setenv("TM_STAGED_KERNEL", flavour)
    else:
        monkeypatch.delenv("TM_STAGED_KERNEL", raising=False)
    what = f"bsp case {i}: k={k} P={P} {strategy} {path} {flavour} mom={mom} lr={lr} mu={mu}"
    W = worker_buffers(P, k, "D2", config=780)
    V = worker_buffers(P, k, "D4", config=781)
    G = worker_buffers(P, k, "D2", config=782)
    Wd, Vd, Gd = to_dev(W), to_dev(V), to_dev(G)
    with tm.Exchanger(P, strategy, size=k, nlocal=k, path=path) as ex:
        for _ in range(2):
            ex.bsp_step(Wd, Vd, Gd, lr, mu, exchange_momentum=mom)
        code, _ = ex.status()
    assert code == tm.TM_OK, what
    ww, vv = W, V
    for _ in range(2):
        ww, vv = bsp_iteration(ww, vv, G, np.float32(lr), np.float32(mu), strategy, exchange_momentum=mom)
    gW, gV = to_host(Wd), to_host(Vd)
    for r in range(k):
        assert_bitwise(gW[r], ww[r], f"{what} w rank {r}")
        assert_bitwise(gV[r], vv[r], f"{what} v rank {r}")


NEASGD = int(os.environ.get("TM_FUZZ_EASGD_CASES", "64"))


@pytest.mark.parametrize("i", range(NEASGD))
def test_fuzz_easgd_bitwise(i):
    """EASGD: random combinations of the centre size
    n (ragged), the number of workers, an arrival order (distinct workers, or
    with repeats), alpha (dyadic 0.5 / 0.5/k or not, 0.3) and the call -- the
    fused round (tm_easgd_round) or one exclusive update per arrival
    (tm_easgd_update_ex) -- on the default stream or a fresh non-blocking
    stream, bitwise against oracle.easgd.easgd_sequence."""
    from oracle.easgd import easgd_sequence
    g = np.random.default_rng([1605, 8325, 781, i])
    n = max(1, int(np.exp(g.uniform(0.0, np.log(1 << 20)))) + int(g.integers(0, 4)))
    nw = int(g.integers(1, 17))
    if g.random() < 0.5:
        order = [int(w) for w in g.permutation(nw)[: int(g.integers(1, nw + 1))]]
    else:
        order = [int(w) for w in g.integers(0, nw, int(g.integers(1, 33)))]
    alpha = float(np.float32(g.choice([0.5, 0.5 / nw, 0.3])))
    call = "round" if g.random() < 0.7 else "updates"
    side = g.random() < 0.5
    what = f"easgd case {i}: n={n} nw={nw} order={order} alpha={alpha} {call} side_stream={side}"
    W = worker_buffers(n, nw, str(g.choice(["D1", "D2", "D3"])), config=790)
    c0 = worker_buffers(n, 1, "D1", config=791)[0]
    Wd, cd = to_dev(W), to_dev([c0])[0]
    st = torch.cuda.Stream() if side else torch.cuda.current_stream()
    st.wait_stream(torch.cuda.current_stream())
    if call == "round":
        tm.tm_easgd_round(Wd, order, cd, alpha, stream=st)
    else:
        for w in order:
            tm.tm_easgd_update_ex(Wd[w], cd, alpha, stream=st)
    st.synchronize()
    ww, cc = easgd_sequence(W, c0, np.float32(alpha), order)
    gW, gc = to_host(Wd), to_host([cd])[0]
    assert_bitwise(gc, cc, f"{what} centre")
    for w in range(nw):
        assert_bitwise(gW[w], ww[w], f"{what} worker {w}")


NGRAPH = int(os.environ.get("TM_FUZZ_GRAPH_CASES", "32"))


@pytest.mark.parametrize("i", range(NGRAPH))
def test_fuzz_graph_replays_bitwise(monkeypatch, i):
    """CUDA-graph capture of a random plan -- 1-4 steps, each a per-rank
    perturbation x_r <- fl(x_r + d_r) followed by a full exchange or a bucket --
    replayed 1-3 times; the epochs and the one-shot kernel's staging parity live
    on the device, so every replay must equal the oracle applied step by step."""
    g = np.random.default_rng([1605, 8325, 782, i])
    k = int(g.integers(2, 9))
    P = max(8, int(np.exp(g.uniform(np.log(8), np.log(1 << 19)))) + int(g.integers(0, 4)))
    strategy = str(g.choice(["asa", "asa16"]))
    path = "direct" if g.random() < 0.3 else "staged"
    flavour = FLAVOURS[int(g.integers(0, len(FLAVOURS)))] if path == "staged" else None
    plan = []
    for _ in range(int(g.integers(1, 5))):
        if g.random() < 0.5:
            off = int(g.integers(0, P // 4)) * 4
            plan.append((off, int(g.integers(0, P - off + 1))))
        else:
            plan.append((0, P))
    replays = int(g.integers(1, 4))
    if flavour:
        monkeypatch.setenv("TM_STAGED_KERNEL", flavour)
    else:
        monkeypatch.delenv("TM_STAGED_KERNEL", raising=False)
    what = f"graph case {i}: k={k} P={P} {strategy} {path} {flavour} plan={plan} replays={replays}"
    X = worker_buffers(P, k, "D2", config=783)
    D = [np.multiply(d, np.float32(1e-3), dtype=np.float32) for d in worker_buffers(P, k, "D1", config=784)]
    bufs, dd = to_dev(X), to_dev(D)
    with tm.Exchanger(P, strategy, size=k, nlocal=k, path=path) as ex:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            ex.exchange(bufs, s)  # eager warm-up call (also part of the expected sequence)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=s):
                for off, cnt in plan:
                    for b, d in zip(bufs, dd):
                        b.add_(d)
                    if off == 0 and cnt == P:
                        ex.exchange(bufs, s)
                    else:
                        ex.exchange_range(bufs, off, cnt, s)
        torch.cuda.current_stream().wait_stream(s)
        for _ in range(replays):
            graph.replay()
        torch.cuda.synchronize()
        code, _ = ex.status()
        got = to_host(bufs)
        del graph
    assert code == tm.TM_OK, what
    want = ox.exchange(X, strategy)
    for _ in range(replays):
        for off, cnt in plan:
            want = [np.add(w, d, dtype=np.float32) for w, d in zip(want, D)]
            if cnt:
                seg = ox.exchange([w[off:off + cnt] for w in want], strategy)
                for r in range(k):
                    want[r][off:off + cnt] = seg[r]
    for r in range(k):
        assert_bitwise(got[r], want[r], f"{what} rank {r}")
