#!/usr/bin/env python
"""Phase breakdown of the staged exchange kernels (tm_set_phase_log), one GPU.

For each staged kernel flavour (TM_STAGED_KERNEL=tma|tmaws|reg|ws, one subprocess
each), k = 8 ranks in one process, AlexNet-sized ASA16, path=staged: the
per-CTA %globaltimer stamps of one exchange (after warm-up) are reduced to the
median over CTAs of each phase's duration and to the span from the first CTA
start to the last CTA end.
"""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NAMES = ["start", "cast", "ready", "reduce", "reduced", "end"]


def child():
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    from paper_1605_08325_b200 import tm
    torch.cuda.set_device(0)
    P, k = 60_965_224, 8
    bufs = [torch.randn(P, device="cuda") * 0.01 for _ in range(k)]
    with tm.Exchanger(P, "asa16", size=k, nlocal=k, path="staged") as ex:
        lay = ex.layout()
        C = lay["ctas_per_rank"]
        log = torch.zeros(k * C * 8, dtype=torch.int64, device="cuda")
        for _ in range(3):
            ex.exchange(bufs)
        tm.tm_set_phase_log(log)
        ex.exchange(bufs)
        torch.cuda.synchronize()
        tm.tm_set_phase_log(None)
        st = log.cpu().numpy().reshape(k * C, 8)[:, :6].astype(np.int64)
    t0 = st[:, 0].min()
    res = {"kernel": ["reg", "tma", "ws", "tmaws"][lay["staged_kernel"]], "ctas": int(k * C),
           "span_us": round((st[:, 5].max() - t0) / 1e3, 1)}
    for i in range(1, 6):
        if st[:, i].max() == 0:
            continue
        prev = i - 1
        while st[:, prev].max() == 0:
            prev -= 1
        d = (st[:, i] - st[:, prev]) / 1e3
        res[f"{NAMES[prev]}->{NAMES[i]}_us_median"] = round(float(np.median(d)), 1)
        res[f"{NAMES[prev]}->{NAMES[i]}_us_max"] = round(float(d.max()), 1)
    print(json.dumps(res))


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        return child()
    for kern in ("tma", "tmaws", "reg", "ws"):
        env = dict(os.environ, TM_STAGED_KERNEL=kern)
        r = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True)
        print(r.stdout.strip() or r.stderr[-2000:])


if __name__ == "__main__":
    main()
