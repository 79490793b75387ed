#!/usr/bin/env python
"""BSP iteration (momentum SGD + exchange, one fused pass on the direct path) at
AlexNet size for k = 2, 4, 8 ranks on one GPU; TM_BSP_TILE overrides the tile.

    python tools/bsp_k.py
"""
import os, sys, torch
sys.path.insert(0, "."); sys.path.insert(0, "tools")
from paper_1605_08325_b200 import tm
from sweep import timeit
P = 60_965_224
torch.cuda.set_device(0)
for k in (2, 4, 8):
    W = [torch.randn(P, device="cuda") * 0.01 for _ in range(k)]
    V = [torch.zeros(P, device="cuda") for _ in range(k)]
    G = [torch.randn(P, device="cuda") * 0.01 for _ in range(k)]
    with tm.Exchanger(P, "asa16", size=k, nlocal=k, path="direct") as ex:
        ms = timeit(lambda: ex.bsp_step(W, V, G, 0.01, 0.9), graph=True)
    print(f"k={k} tile={os.environ.get('TM_BSP_TILE','512')} {ms*1e3:.1f} us frac {20.0*P*k/(ms*1e-3)/1e9/6553.9:.3f}")
    del W, V, G
    torch.cuda.empty_cache()
