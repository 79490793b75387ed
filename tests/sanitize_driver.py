#!/usr/bin/env python
"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
every kernel of libtm.so on small, ragged sizes, checked against the oracle so
a sanitizer run is also a parity run.

    compute-sanitizer --tool memcheck python tests/sanitize_driver.py
"""

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import exchange as ox  # noqa: E402  (test infrastructure: parity of the run)
from oracle.easgd import easgd_sequence, easgd_update  # noqa: E402
from paper_1605_08325_b200 import tm  # noqa: E402
from paper_1605_08325_b200.inputs import worker_buffers  # noqa: E402


def check(a, b, what):
    if not np.array_equal(np.asarray(a, np.float32).view(np.uint32), np.asarray(b, np.float32).view(np.uint32)):
        raise SystemExit(f"MISMATCH {what}")


def main():
    torch.cuda.set_device(0)
    n_ok = 0
    for k, P in ((2, 5003), (3, 20011), (8, 40961)):
        for strategy in ("asa16", "asa", "ar"):
            for path in ("staged", "direct"):
                X = worker_buffers(P, k, "D2", config=70)
                bufs = [torch.from_numpy(x).cuda() for x in X]
                with tm.Exchanger(P, strategy, size=k, nlocal=k, path=path) as ex:
                    ex.exchange(bufs)
                    ex.exchange(bufs)
                    code, _ = ex.status()
                assert code == 0, code
                want = ox.exchange(ox.exchange(X, strategy), strategy)
                for r in range(k):
                    check(bufs[r].cpu().numpy(), want[r], f"{strategy} {path} k={k} P={P}")
                n_ok += 1
    W = worker_buffers(30011, 4, "D1", config=71)
    c = worker_buffers(30011, 1, "D1", config=72)[0]
    Wd = [torch.from_numpy(w).cuda() for w in W]
    cd = torch.from_numpy(c).cuda()
    tm.tm_easgd_round(Wd, [2, 0, 3, 1], cd, 0.125)
    tm.tm_easgd_round(Wd, [1, 1, 0], cd, 0.125)
    tm.tm_easgd_update_ex(Wd[0], cd, 0.3)
    tm.tm_easgd_update_ex(Wd[1], cd, 0.3, concurrent=True)
    ws, cc = easgd_sequence(W, c, 0.125, [2, 0, 3, 1])
    ws, cc = easgd_sequence(ws, cc, 0.125, [1, 1, 0])
    ws[0], cc = easgd_update(ws[0], cc, 0.3)
    ws[1], cc = easgd_update(ws[1], cc, 0.3)
    check(cd.cpu().numpy(), cc, "easgd centre")
    for r in range(4):
        check(Wd[r].cpu().numpy(), ws[r], f"easgd worker {r}")
    from oracle.bsp import bsp_iteration
    for path in ("direct", "staged"):  # BSP step: TMA-engine one pass / step fused into the pre-cast
        k, P = 3, 20011
        Wb = worker_buffers(P, k, "D2", config=73)
        Vb = worker_buffers(P, k, "D4", config=74)
        Gb = worker_buffers(P, k, "D2", config=75)
        Wt, Vt, Gt = ([torch.from_numpy(a).cuda() for a in arrs] for arrs in (Wb, Vb, Gb))
        with tm.Exchanger(P, "asa16", size=k, nlocal=k, path=path) as ex:
            ex.bsp_step(Wt, Vt, Gt, 0.01, 0.9, exchange_momentum=True)
        ww, vv = bsp_iteration(Wb, Vb, Gb, 0.01, 0.9, "asa16", exchange_momentum=True)
        for r in range(k):
            check(Wt[r].cpu().numpy(), ww[r], f"bsp w {path}")
            check(Vt[r].cpu().numpy(), vv[r], f"bsp v {path}")
        n_ok += 1
    # round 2: exact concurrent EASGD (CAS loop), and bucket exchanges under a CTA budget
    W2 = worker_buffers(20011, 2, "D1", config=76)
    c2 = worker_buffers(20011, 1, "D1", config=77)[0]
    W2d = [torch.from_numpy(w).cuda() for w in W2]
    c2d = torch.from_numpy(c2).cuda()
    tm.tm_easgd_update_ex(W2d[0], c2d, 0.25, concurrent="exact")
    w0, cc2 = easgd_update(W2[0], c2, 0.25)
    check(c2d.cpu().numpy(), cc2, "easgd exact centre")
    check(W2d[0].cpu().numpy(), w0, "easgd exact worker")
    for path in ("direct", "staged"):
        k, P = 3, 30011
        X = worker_buffers(P, k, "D2", config=78)
        bufs = [torch.from_numpy(x).cuda() for x in X]
        with tm.Exchanger(P, "asa16", size=k, nlocal=k, path=path) as ex:
            tm.tm_set_range_ctas(2)
            ex.exchange_range(bufs, 12000, P - 12000)
            ex.exchange_range(bufs, 0, 12000)
        want = ox.exchange(X, "asa16")
        for r in range(k):
            check(bufs[r].cpu().numpy(), want[r], f"budget range {path}")
        n_ok += 1
    x = torch.randn(100003, device="cuda")
    h = tm.tm_cast_rn16(x)
    torch.cuda.synchronize()
    print(f"sanitize driver ok: {n_ok} exchanges + easgd + cast, all bitwise == oracle")


if __name__ == "__main__":
    main()
