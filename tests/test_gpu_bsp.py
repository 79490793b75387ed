"""GPU parity of tm_bsp_step(_group) (momentum SGD + exchange) against
oracle/bsp.py, both data paths, with and without momentum exchange."""

import numpy as np
import pytest
import torch

from gpu_helpers import assert_bitwise, to_dev, to_host
from oracle.bsp import bsp_iteration
from paper_1605_08325_b200 import tm
from paper_1605_08325_b200.inputs import worker_buffers

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mom", [False, True])
@pytest.mark.parametrize("path", ["staged", "direct"])
@pytest.mark.parametrize("strategy", ["asa16", "asa", "ar"])
def test_bsp_step_group_bitwise(strategy, path, mom):
    lr, mu = 0.01, 0.9
    for k, P in ((2, 9), (3, 4099), (8, 300_007)):
        W = worker_buffers(P, k, "D2", config=100)
        V = worker_buffers(P, k, "D4", config=101)
        G = worker_buffers(P, k, "D2", config=102)
        Wd, Vd, Gd = to_dev(W), to_dev(V), to_dev(G)
        with tm.Exchanger(P, strategy, size=k, nlocal=k, path=path) as ex:
            for _ in range(2):  # two iterations: state carries over
                ex.bsp_step(Wd, Vd, Gd, lr, mu, exchange_momentum=mom)
            code, _ = ex.status()
        assert code == tm.TM_OK
        ww, vv = W, V
        for _ in range(2):
            ww, vv = bsp_iteration(ww, vv, G, lr, mu, strategy, exchange_momentum=mom)
        gW, gV = to_host(Wd), to_host(Vd)
        for r in range(k):
            assert_bitwise(gW[r], ww[r], f"w {strategy} {path} mom={mom} k={k} P={P} r={r}")
            assert_bitwise(gV[r], vv[r], f"v {strategy} {path} mom={mom} k={k} P={P} r={r}")


def test_bsp_step_rejects_sum_mode():
    P = 1024
    with tm.Exchanger(P, "asa", size=2, nlocal=2, op="sum"):
        b = [torch.zeros(P, device="cuda") for _ in range(2)]
        with pytest.raises(tm.TmError) as e:
            tm.tm_bsp_step_group(b, b, b, 0.1, 0.9)
        assert e.value.code == tm.TM_E_ARG


@pytest.mark.parametrize("kernel", ["reg", "tma", "ws", "tmaws", "oneshot", "ll", "ll2"])
@pytest.mark.parametrize("unfused", ["0", "1"])
def test_bsp_staged_flavours_bitwise(monkeypatch, kernel, unfused):
    """Single-process group on the staged path, every staged kernel flavour, with
    the step fused into the pre-cast (default) and as a separate SGD kernel
    (TM_BSP_UNFUSED=1): ragged P (P % 4 = 3, several tiles), both strategies."""
    monkeypatch.setenv("TM_STAGED_KERNEL", kernel)
    monkeypatch.setenv("TM_BSP_UNFUSED", unfused)
    lr, mu = 0.05, 0.9
    for strategy, mom, k, P in (("asa16", False, 4, 1_000_003), ("asa", True, 3, 70_003),
                                ("asa16", True, 8, 20_483)):
        W = worker_buffers(P, k, "D1", config=110)
        V = worker_buffers(P, k, "D4", config=111)
        G = worker_buffers(P, k, "D2", config=112)
        Wd, Vd, Gd = to_dev(W), to_dev(V), to_dev(G)
        with tm.Exchanger(P, strategy, size=k, nlocal=k, path="staged") as ex:
            assert ex.layout()["staged_kernel"] == {"reg": 0, "tma": 1, "ws": 2, "tmaws": 3, "oneshot": 4, "ll": 5, "ll2": 6}[kernel]
            for _ in range(3):
                ex.bsp_step(Wd, Vd, Gd, lr, mu, exchange_momentum=mom)
            code, _ = ex.status()
        assert code == tm.TM_OK
        ww, vv = W, V
        for _ in range(3):
            ww, vv = bsp_iteration(ww, vv, G, lr, mu, strategy, exchange_momentum=mom)
        gW, gV = to_host(Wd), to_host(Vd)
        for r in range(k):
            assert_bitwise(gW[r], ww[r], f"w {kernel} {strategy} k={k} P={P} r={r}")
            assert_bitwise(gV[r], vv[r], f"v {kernel} {strategy} k={k} P={P} r={r}")


def test_bsp_staged_status_overflow(monkeypatch):
    """The fused pre-cast screens w' = w + v' (not w): a step that pushes a weight
    past the binary16 range sets TM_BIT_OVERFLOW16."""
    P, k = 4096, 2
    W = [np.zeros(P, np.float32) for _ in range(k)]
    V = [np.zeros(P, np.float32) for _ in range(k)]
    G = [np.zeros(P, np.float32) for _ in range(k)]
    G[1][777] = np.float32(-1e6)  # v' = 0.1 * 1e6 -> w' = 1e5 > 65504
    Wd, Vd, Gd = to_dev(W), to_dev(V), to_dev(G)
    with tm.Exchanger(P, "asa16", size=k, nlocal=k, path="staged") as ex:
        ex.bsp_step(Wd, Vd, Gd, 0.1, 0.9)
        code, bits = ex.status()
    assert bits & tm.TM_BIT_OVERFLOW16, (code, bits)


@pytest.mark.parametrize("path", ["direct", "staged"])
def test_bsp_full_size_sampled(path):
    """AlexNet size, k = 8 (the launch configuration the BSP sweep times): sampled
    elements and the tail against oracle/bsp.py (elementwise, so the oracle runs
    on the sampled columns)."""
    from paper_1605_08325_b200.inputs import WORKLOADS
    P, k = WORKLOADS["alexnet"], 8
    W = worker_buffers(P, k, "D2", config=120)
    V = worker_buffers(P, k, "D4", config=121)
    G = worker_buffers(P, k, "D2", config=122)
    idx = np.unique(np.concatenate([np.random.default_rng(9).integers(0, P, 100_000),
                                    np.arange(P - 300, P)]))
    want_w, want_v = bsp_iteration([w[idx] for w in W], [v[idx] for v in V], [g[idx] for g in G],
                                   0.01, 0.9, "asa16")
    Wd, Vd, Gd = to_dev(W), to_dev(V), to_dev(G)
    del W, V, G
    with tm.Exchanger(P, "asa16", size=k, nlocal=k, path=path) as ex:
        ex.bsp_step(Wd, Vd, Gd, 0.01, 0.9)
        code, _ = ex.status()
    assert code == tm.TM_OK
    ti = torch.from_numpy(idx).cuda()
    for r in (0, 5, 7):
        assert_bitwise(Wd[r][ti].cpu().numpy(), want_w[r], f"w {path} rank {r}")
        assert_bitwise(Vd[r][ti].cpu().numpy(), want_v[r], f"v {path} rank {r}")
    del Wd, Vd, Gd
    torch.cuda.empty_cache()
