"""Reuse protocol under load: 10^4 back-to-back staged exchanges
in one process (k ranks' CTAs on one GPU, flags at GPU scope, device-side epochs
across captured-graph replays), each after a per-rank fp32 perturbation, for
every staged kernel flavour.  The method is elementwise, so the oracle replays
the whole sequence on sampled columns (plus the tail) and must agree bitwise."""

import numpy as np
import pytest
import torch

from gpu_helpers import assert_bitwise
from oracle import exchange as ox
from paper_1605_08325_b200 import tm
from paper_1605_08325_b200.inputs import worker_buffers

pytestmark = pytest.mark.gpu

N_EXCHANGES = 10_000
PER_GRAPH = 100


@pytest.mark.parametrize("kernel", ["reg", "tma", "ws", "tmaws", "oneshot", "ll", "ll2"])
@pytest.mark.parametrize("strategy", ["asa16", "asa"])
def test_ten_thousand_exchanges(monkeypatch, kernel, strategy):
    monkeypatch.setenv("TM_STAGED_KERNEL", kernel)
    k, P = 3, 3 * 8192 + 5  # several CTAs per rank, ragged tail
    X = worker_buffers(P, k, "D2", config=140)
    D = [d * np.float32(1e-3) for d in worker_buffers(P, k, "D1", config=141)]
    bufs = [torch.from_numpy(x).cuda() for x in X]
    deltas = [torch.from_numpy(d).cuda() for d in D]
    with tm.Exchanger(P, strategy, size=k, nlocal=k, path="staged") as ex:
        assert ex.layout()["ctas_per_rank"] > 1
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        # the perturbation alternates in sign so the values stay in range and no
        # exchange reaches a rounding fixed point
        with torch.cuda.stream(s):
            for b, d in zip(bufs, deltas):  # one exchange outside the graph
                b.add_(d)
            ex.exchange(bufs, s)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for j in range(PER_GRAPH):
                    for b, d in zip(bufs, deltas):
                        b.sub_(d) if j % 2 else b.add_(d)
                    ex.exchange(bufs, s)
        torch.cuda.current_stream().wait_stream(s)
        for _ in range(N_EXCHANGES // PER_GRAPH):
            g.replay()
        torch.cuda.synchronize()
        code, bits = ex.status()
    assert code == tm.TM_OK, (code, bits)
    idx = np.unique(np.concatenate([np.random.default_rng(3).integers(0, P, 96), np.arange(P - 5, P)]))
    cols = np.stack([x[idx] for x in X])
    dcols = np.stack([d[idx] for d in D])
    signs = [+1] + [(-1 if j % 2 else 1) for j in range(PER_GRAPH)] * (N_EXCHANGES // PER_GRAPH)
    for sg in signs:  # after each exchange every rank holds the same average
        pert = np.add(cols, dcols, dtype=np.float32) if sg > 0 else np.subtract(cols, dcols, dtype=np.float32)
        avg = ox.element_average(pert, strategy)
        cols = np.stack([avg] * k)
    ti = torch.from_numpy(idx).cuda()
    for r in range(k):
        assert_bitwise(bufs[r][ti].cpu().numpy(), cols[r], f"{kernel} {strategy} rank {r}")
