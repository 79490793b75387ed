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
