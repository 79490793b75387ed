#!/usr/bin/env python
"""The allgather decision step (north star: NCCL allgather "only where it
measures faster"): read the bench lines tools/multigpu_eval.sh wrote for every
allgather mode (sm / ce / nccl) at each N and workload, keep the fastest mode
per (k, L), and write the rule table the library reads at init through
TM_AG_TABLE ("k L_max mode" per line; a mode covers segment lengths up to the
midpoint to the next measured L).

    python tools/ag_decide.py [gpurun_out/multigpu] > profiles/ag_table.txt
"""
import glob
import json
import os
import re
import sys


def main():
    d = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/multigpu"
    best = {}  # (k, L) -> (ms, mode)
    for f in glob.glob(os.path.join(d, "bench_n*_ag*.json")):
        m = re.search(r"_ag(sm|ce|nccl)", f)
        try:
            line = json.loads(open(f).read().strip().splitlines()[-1])
        except Exception:
            continue
        if not (line.get("parity") or {}).get("parity"):
            continue  # only modes whose results were checked
        if line["config"].get("staged_kernel") == "tm_exchange_oneshot_kernel":
            continue  # no allgather phase: the mode does not apply
        k, L, ms = line["config"]["k"], line["config"]["seg_len"], line["ms_per_step"]
        cur = best.get((k, L))
        if cur is None or ms < cur[0]:
            best[(k, L)] = (ms, m.group(1))
    print("# k L_max mode  (fastest measured allgather per (k, L); tools/ag_decide.py)")
    for k in sorted({k for k, _ in best}):
        Ls = sorted(L for kk, L in best if kk == k)
        for i, L in enumerate(Ls):
            lmax = (L + Ls[i + 1]) // 2 if i + 1 < len(Ls) else 1 << 62
            print(k, lmax, best[(k, L)][1], f"# measured at L={L}: {best[(k, L)][0]:.4f} ms")


if __name__ == "__main__":
    main()
