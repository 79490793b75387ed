"""The staged path's allgather outside the kernel (tm_allgather, SURVEY 8(a)
a6): copy engines (TM_AG_CE) and NCCL (TM_AG_NCCL) gather the averaged
segments after the kernel's reduced barrier; results must stay bitwise those of
the fused SM pull and of the oracle."""

import os

import numpy as np
import pytest
import torch

from gpu_helpers import assert_bitwise, to_dev, to_host
from oracle import exchange as ox
from oracle.bsp import bsp_iteration
from paper_1605_08325_b200 import tm
from paper_1605_08325_b200.inputs import worker_buffers

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kernel", ["tma", "ws", "reg", "tmaws"])
@pytest.mark.parametrize("strategy", ["asa16", "asa"])
def test_copy_engine_allgather_bitwise(monkeypatch, kernel, strategy):
    monkeypatch.setenv("TM_STAGED_KERNEL", kernel)
    for k, P, dist in ((2, 9, "D6"), (3, 100_003, "D2"), (8, 1_000_003, "D4"), (5, 4_099, "D1")):
        X = worker_buffers(P, k, dist, config=130)
        bufs = to_dev(X)
        with tm.Exchanger(P, strategy, size=k, nlocal=k, path="staged", allgather="ce") as ex:
            assert ex.layout()["allgather"] == tm.TM_AG_CE
            for _ in range(2):  # reuse of staging across exchanges
                ex.exchange(bufs)
            code, _ = ex.status()
        want = ox.exchange(ox.exchange(X, strategy), strategy)
        got = to_host(bufs)
        for r in range(k):
            assert_bitwise(got[r], want[r], f"{kernel} {strategy} k={k} P={P} r={r}")
        assert code in (tm.TM_OK, tm.TM_E_NONFINITE, tm.TM_E_OVERFLOW16)


def test_copy_engine_allgather_ranges_bsp_and_graph():
    """Bucketed ranges, the fused BSP step and CUDA-graph capture with the copy
    engines doing the allgather."""
    k, P = 4, 300_007
    X = worker_buffers(P, k, "D2", config=131)
    bufs = to_dev(X)
    with tm.Exchanger(P, "asa16", size=k, nlocal=k, path="staged", allgather="ce") as ex:
        b1, b2 = P // 3 // 4 * 4, 2 * P // 3 // 4 * 4
        for off, n in ((b2, P - b2), (b1, b2 - b1), (0, b1)):
            ex.exchange_range(bufs, off, n)
        want = ox.exchange(X, "asa16")
        for r, g in enumerate(to_host(bufs)):
            assert_bitwise(g, want[r], f"range r={r}")
        # graph capture of one exchange, replayed twice
        g2 = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(g2, stream=s):
                ex.exchange(bufs, s)
        torch.cuda.current_stream().wait_stream(s)
        g2.replay()
        g2.replay()
        torch.cuda.synchronize()
        want = ox.exchange(ox.exchange(want, "asa16"), "asa16")
        for r, g in enumerate(to_host(bufs)):
            assert_bitwise(g, want[r], f"graph r={r}")
        W = worker_buffers(P, k, "D2", config=132)
        V = worker_buffers(P, k, "D4", config=133)
        G = worker_buffers(P, k, "D2", config=134)
        Wd, Vd, Gd = to_dev(W), to_dev(V), to_dev(G)
        ex.bsp_step(Wd, Vd, Gd, 0.01, 0.9, exchange_momentum=True)
        ww, vv = bsp_iteration(W, V, G, 0.01, 0.9, "asa16", exchange_momentum=True)
        for r in range(k):
            assert_bitwise(to_host([Wd[r]])[0], ww[r], f"bsp w r={r}")
            assert_bitwise(to_host([Vd[r]])[0], vv[r], f"bsp v r={r}")


def test_allgather_mode_errors():
    with tm.Exchanger(1024, "asa16", size=2, nlocal=2) as ex:
        assert ex.layout()["allgather"] == tm.TM_AG_SM
        with pytest.raises(tm.TmError) as e:
            tm.tm_set_allgather("nccl")  # no communicator in a single-process group
        assert e.value.code == tm.TM_E_NCCL
        with pytest.raises(tm.TmError) as e:
            tm.tm_set_allgather(7)
        assert e.value.code == tm.TM_E_ARG
        tm.tm_set_allgather("ce")
        assert ex.layout()["allgather"] == tm.TM_AG_CE
        tm.tm_set_allgather("sm")
