"""GPU parity of the parallel loading process (tm_loader_*, PAPER Alg. 1)
against oracle/loader.py, protocol replay, error reporting and overlap."""

import os
import time

import numpy as np
import pytest
import torch

from gpu_helpers import assert_bitwise
from oracle import loader as ol
from paper_1605_08325_b200 import tm

pytestmark = pytest.mark.gpu

N, C, H, W, CH, CW = 4, 3, 40, 48, 32, 40


def _files(tmp_path, count, seed=0):
    g = np.random.default_rng([1605, 8325, 60, seed])
    paths, raws = [], {}
    for i in range(count):
        raw = g.integers(0, 256, (N, C, H, W)).astype(np.uint8)
        p = str(tmp_path / f"batch_{i:04d}.pxb")
        tm.write_batch_file(p, raw)
        paths.append(p)
        raws[p] = raw
    mean = g.uniform(0, 255, (C, H, W)).astype(np.float32)
    return paths, raws, mean


def test_alg1_sequence_bitwise(tmp_path):
    """train f0 f1 f2 | val v0 v1 | stop: the trainer receives the batches Alg. 1
    delivers (deliveries()), each bitwise equal to the oracle's preprocessing
    with the load index the loader used."""
    paths, raws, mean = _files(tmp_path, 6)
    f0, f1, f2, v0, v1, _ = paths
    msgs = [("train", None), ("file", f0), ("file", f1), ("file", f2), ("val", None),
            ("file", v0), ("file", v1), ("stop", None)]
    expected = ol.deliveries(msgs)
    assert [e[0] for e in expected] == [f0, f1, v0]
    seed = 20260
    got = []
    # replay deterministically: one loader, messages interleaved with waits
    x = torch.zeros(N * C * CH * CW, device="cuda")
    with tm.Loader(N, C, H, W, CH, CW, mean, x, seed=seed) as L:
        L.send("train"); L.send("file", f0)
        L.send("file", f1); L.wait(10_000); got.append(x.clone())
        L.send("file", f2); L.wait(10_000); got.append(x.clone())
        L.send("val"); L.send("file", v0)
        L.send("file", v1); L.wait(10_000); got.append(x.clone())
        L.send("stop")
    for (name, mode, idx), t in zip(expected, got):
        want = ol.preprocess(raws[name], mean, CH, CW, mode, seed, idx)
        assert_bitwise(t.cpu().numpy(), want.reshape(-1), f"{name} {mode} load {idx}")


def test_missing_file_reports_io_error(tmp_path):
    paths, raws, mean = _files(tmp_path, 1)
    x = torch.zeros(N * C * CH * CW, device="cuda")
    with tm.Loader(N, C, H, W, CH, CW, mean, x) as L:
        L.send("train")
        L.send("file", str(tmp_path / "does_not_exist.pxb"))
        L.send("file", paths[0])
        with pytest.raises(tm.TmError) as e:
            L.wait(10_000)
        assert e.value.code == tm.TM_E_IO


def test_wrong_shape_and_protocol_errors(tmp_path):
    paths, raws, mean = _files(tmp_path, 1)
    x = torch.zeros(N * C * CH * CW, device="cuda")
    with tm.Loader(N, C, H, W, CH - 2, CW, mean, x[: N * C * (CH - 2) * CW]) as L:
        L.send("file", paths[0])  # a filename where Alg. 1 expects a mode
        with pytest.raises(tm.TmError) as e:
            L.wait(10_000)
        assert e.value.code == tm.TM_E_ARG
    bad = str(tmp_path / "bad.pxb")
    tm.write_batch_file(bad, np.zeros((N, C, H, W + 1), np.uint8))
    with tm.Loader(N, C, H, W, CH, CW, mean, x) as L:
        L.send("val"); L.send("file", bad); L.send("file", paths[0])
        with pytest.raises(tm.TmError) as e:
            L.wait(10_000)
        assert e.value.code == tm.TM_E_IO


def test_loading_overlaps_training(tmp_path):
    """with per-batch load time L and compute time T = L, n pipelined
    iterations take <= 0.75 n (L + T) + C.  L is measured (loader alone), the
    trainer's compute is a host sleep of the same length."""
    n_b, c, h, w, ch, cw = 64, 3, 256, 256, 227, 227
    g = np.random.default_rng(3)
    mean = g.uniform(0, 255, (c, h, w)).astype(np.float32)
    paths = []
    for i in range(4):
        p = str(tmp_path / f"big_{i}.pxb")
        tm.write_batch_file(p, g.integers(0, 256, (n_b, c, h, w)).astype(np.uint8))
        paths.append(p)
    files = [paths[i % 4] for i in range(24)]
    x = torch.zeros(n_b * c * ch * cw, device="cuda")

    def run(compute_s):
        with tm.Loader(n_b, c, h, w, ch, cw, mean, x, seed=1) as L:
            t0 = time.perf_counter()
            L.send("train"); L.send("file", files[0])
            for f in files[1:]:
                L.send("file", f)   # training on the previous input_x is done
                L.wait(60_000)      # the next batch is in input_x
                time.sleep(compute_s)
            return time.perf_counter() - t0

    run(0.0)  # warm the page cache
    load = run(0.0) / (len(files) - 1)
    total = run(load)
    n = len(files) - 1
    assert total <= 0.75 * n * (2 * load) + 0.05, (total, load)


def test_file_message_waits_for_trainer_stream(tmp_path):
    """A FILE message releases the loaded batch into input_x (Alg. 1); the
    trainer's kernels that still read the previous batch may be queued on its
    stream when the message is sent, so the loader's copy waits for the work
    enqueued on that stream before the send (tm_loader_send_after).  Here the
    trainer's stream sleeps ~0.1 s and then snapshots input_x: the snapshot must
    be the PREVIOUS batch, not the one the message releases."""
    paths, raws, mean = _files(tmp_path, 3)
    f0, f1, f2 = paths
    x = torch.zeros(N * C * CH * CW, device="cuda")
    s = torch.cuda.Stream()
    with tm.Loader(N, C, H, W, CH, CW, mean, x, seed=5) as L:
        L.send("train"); L.send("file", f0)
        L.send("file", f1); L.wait(10_000)  # input_x = batch f0 (load 0)
        want0 = x.clone()
        torch.cuda.synchronize()
        with torch.cuda.stream(s):
            torch.cuda._sleep(200_000_000)  # the trainer is still busy ...
            snap = x.clone()                # ... and then reads input_x
            L.send("file", f2, stream=s)    # releases batch f1 into input_x
        L.wait(10_000)
        torch.cuda.synchronize()
        after = x.clone()
    assert_bitwise(snap.cpu().numpy(), want0.cpu().numpy(), "trainer's read of the previous batch")
    want1 = ol.preprocess(raws[f1], mean, CH, CW, "train", 5, 1)
    assert_bitwise(after.cpu().numpy(), want1.reshape(-1), "released batch")


@pytest.mark.parametrize("i", range(16))
def test_fuzz_loader_sequences_bitwise(tmp_path, i):
    """Seeded random Alg. 1 sessions: random batch geometry (odd
    sizes, crop up to the full image), 2-4 mode segments (train / val) of 1-4
    files each, the trainer waiting for every delivery the state machine makes
    (oracle deliveries()) and reading input_x after it; every delivered batch
    bitwise equal to oracle.loader.preprocess with the loader's load index."""
    g = np.random.default_rng([1605, 8325, 61, i])
    n, c = int(g.integers(1, 6)), int(g.integers(1, 4))
    h, w = int(g.integers(1, 40)), int(g.integers(1, 40))
    ch, cw = int(g.integers(1, h + 1)), int(g.integers(1, w + 1))
    seed = int(g.integers(0, 1 << 62))
    mean = g.uniform(0, 255, (c, h, w)).astype(np.float32)
    msgs, raws = [], {}
    for s in range(int(g.integers(2, 5))):
        msgs.append((str(g.choice(["train", "val"])), None))
        for f in range(int(g.integers(1, 5))):
            p = str(tmp_path / f"b{s}_{f}.pxb")
            raws[p] = g.integers(0, 256, (n, c, h, w)).astype(np.uint8)
            tm.write_batch_file(p, raws[p])
            msgs.append(("file", p))
    msgs.append(("stop", None))
    expected = ol.deliveries(msgs)
    x = torch.zeros(n * c * ch * cw, device="cuda")
    got = []
    with tm.Loader(n, c, h, w, ch, cw, mean, x, seed=seed) as L:
        prev_file = False
        for kind, name in msgs:
            L.send(kind, name)
            if kind == "file" and prev_file:  # a FILE after a loaded file delivers it
                L.wait(10_000)
                got.append(x.clone())
            prev_file = kind == "file"
    assert len(got) == len(expected), (len(got), expected)
    for (name, mode, idx), t in zip(expected, got):
        want = ol.preprocess(raws[name], mean, ch, cw, mode, seed, idx)
        assert_bitwise(t.cpu().numpy(), want.reshape(-1), f"case {i} {name} {mode} load {idx}")
