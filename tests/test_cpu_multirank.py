"""World-size-2 gloo tests (CPU) of the host-side multi-rank logic: the bootstrap
blob all-gather, bench.py's max-over-ranks timing and whole-job value, and the
reference arm's rank-0-only output under torchrun."""

import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


WORKER = r'''
import json, os, sys
sys.path.insert(0, sys.argv[1])
import torch.distributed as dist
dist.init_process_group("gloo")
r, n = dist.get_rank(), dist.get_world_size()
from paper_1605_08325_b200 import tm
import bench
blob = bytes([r]) * 512
blobs = tm.gather_blobs(blob, n)
t = bench.reduce_max(1.5 + r, "cpu")
v = bench.job_value(4.0 * 1000, n, t)
json.dump({"order": [b[0] for b in blobs], "lens": [len(b) for b in blobs], "max": t, "value": v},
          open(os.path.join(sys.argv[2], f"r{r}.json"), "w"))
try:
    tm.gather_blobs(blob, n + 1)
    bad = False
except ValueError:
    bad = True
json.dump(bad, open(os.path.join(sys.argv[2], f"bad{r}.json"), "w"))
dist.destroy_process_group()
'''


def _launch(n, argv, tmp_path, extra_env=None):
    port = _port()
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(n), LOCAL_RANK=str(r),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), **(extra_env or {}))
        procs.append(subprocess.Popen(argv, env=env, stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                      text=True))
    outs = []
    for p in procs:
        o, e = p.communicate(timeout=300)
        outs.append((p.returncode, o, e))
    return outs


def test_bootstrap_gather_and_max_over_ranks(tmp_path):
    script = tmp_path / "w.py"
    script.write_text(WORKER)
    outs = _launch(2, [sys.executable, str(script), ROOT, str(tmp_path)], tmp_path)
    for rc, o, e in outs:
        assert rc == 0, e[-2000:]
    for r in range(2):
        d = json.load(open(tmp_path / f"r{r}.json"))
        assert d["order"] == [0, 1] and d["lens"] == [512, 512]
        assert d["max"] == 2.5  # max over ranks, identical on every rank
        assert abs(d["value"] - 4.0 * 1000 * 2 / 2.5e-3 / 1e9) < 1e-12
        assert json.load(open(tmp_path / f"bad{r}.json")) is True


def test_reference_arm_rank0_only(tmp_path):
    """Under torchrun only rank 0 runs the oracle and prints one JSON line; the
    other rank exits 0 without output."""
    outs = _launch(2, [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                       "--gpus", "2", "--steps", "2", "--warmup", "1", "--workload", "1m"],
                   tmp_path, extra_env={"REF_BUDGET_S": "2"})
    (rc0, o0, e0), (rc1, o1, e1) = outs
    assert rc0 == 0 and rc1 == 0, (e0[-1000:], e1[-1000:])
    assert o1.strip() == ""
    lines = [l for l in o0.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["config"]["k"] == 2
    assert d["unit"] == "GB/s" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0


PARITY_WORKER = r'''
import json, os, sys
sys.path.insert(0, sys.argv[1])
import numpy as np
import torch.distributed as dist
dist.init_process_group("gloo")
r, n = dist.get_rank(), dist.get_world_size()
import bench
from oracle import exchange as ox
from paper_1605_08325_b200.inputs import worker_buffer
P = 20_011
idx = bench.sample_indices(P)
# what every rank's GPU result would hold at the sampled indices (the oracle's
# average of all ranks' seeded inputs); rank 1 flips one bit when asked to
vals = np.stack([worker_buffer(P, "D2", q, config=3)[idx] for q in range(n)])
mine = ox.element_average(vals, "asa16")
if r == 1 and sys.argv[3] == "corrupt":
    mine.view(np.uint32)[5] ^= 1
got = [None] * n
dist.all_gather_object(got, mine)
if r == 0:
    res = bench.check_sample("asa16", "D2", P, n, idx, got)
    json.dump(res, open(os.path.join(sys.argv[2], "parity.json"), "w"))
dist.barrier()
dist.destroy_process_group()
'''


@pytest.mark.parametrize("mode", ["clean", "corrupt"])
def test_multi_rank_parity_check_flow(tmp_path, mode):
    """bench.py's N>1 parity path over gloo, world size 2: every rank's sampled
    outputs are all-gathered to rank 0, which regenerates every rank's seeded
    input and checks them against the oracle's per-element definition; a single
    flipped bit on rank 1 fails that rank and the cross-rank identity."""
    script = tmp_path / "p.py"
    script.write_text(PARITY_WORKER)
    outs = _launch(2, [sys.executable, str(script), ROOT, str(tmp_path), mode], tmp_path)
    for rc, o, e in outs:
        assert rc == 0, e[-2000:]
    res = json.load(open(tmp_path / "parity.json"))
    if mode == "clean":
        assert res["parity"] and res["per_rank"] == [True, True] and res["cross_rank_identical"]
    else:
        assert not res["parity"] and res["per_rank"] == [True, False] and not res["cross_rank_identical"]
