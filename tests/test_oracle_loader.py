"""Pins for oracle/loader.py (CPU only)."""

import os

import numpy as np
import pytest

from oracle import loader as ol

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "splitmix64.txt")


def test_splitmix64_published_outputs():
    rows = [l.split() for l in open(GOLDEN) if l.strip() and not l.startswith("#")]
    assert len(rows) == 6
    for seed, idx, want in rows:
        x = int(seed)
        for _ in range(int(idx)):
            x = (x + 0x9E3779B97F4A7C15) & ol.MASK
        assert ol.splitmix64(x) == int(want)


def _batch(n=3, c=2, h=9, w=11, seed=0):
    g = np.random.default_rng([1605, 8325, 7, seed])
    raw = g.integers(0, 256, (n, c, h, w)).astype(np.uint8)
    mean = g.uniform(0, 255, (c, h, w)).astype(np.float32)
    return raw, mean


def test_mean_equal_to_data_gives_zeros():
    # mean = data (constant batch) -> all-zero output
    raw = np.full((2, 3, 8, 8), 17, np.uint8)
    mean = np.full((3, 8, 8), 17.0, np.float32)
    for mode in ("train", "val"):
        out = ol.preprocess(raw, mean, 5, 6, mode, seed=3, file_index=4)
        assert out.shape == (2, 3, 5, 6) and np.all(out == 0)


def test_val_is_deterministic_centre_crop():
    # val mode is deterministic (centre crop, no mirror)
    raw, mean = _batch()
    a = ol.preprocess(raw, mean, 5, 7, "val", seed=1, file_index=0)
    b = ol.preprocess(raw, mean, 5, 7, "val", seed=99, file_index=12)
    assert np.array_equal(a, b)
    oy, ox = (9 - 5) // 2, (11 - 7) // 2
    want = raw[:, :, oy:oy + 5, ox:ox + 7].astype(np.float32) - mean[None, :, oy:oy + 5, ox:ox + 7]
    assert np.array_equal(a, want.astype(np.float32))


def test_train_matches_element_loop():
    """Element-by-element Python loop over the definition (mean subtracted at the
    source pixel, then cropped and mirrored)."""
    raw, mean = _batch(n=4)
    n, c, h, w = raw.shape
    ch, cw = 6, 5
    out = ol.preprocess(raw, mean, ch, cw, "train", seed=11, file_index=2)
    params = ol.crop_params(n, h, w, ch, cw, "train", 11, 2)
    for b in range(n):
        oy, ox, mir = params[b]
        assert 0 <= oy <= h - ch and 0 <= ox <= w - cw and mir in (0, 1)
        for k in range(c):
            for y in range(ch):
                for x in range(cw):
                    xs = cw - 1 - x if mir else x
                    want = np.float32(np.float32(raw[b, k, oy + y, ox + xs]) - mean[k, oy + y, ox + xs])
                    assert out[b, k, y, x] == want


def test_crop_params_cover_range_and_mirror_half():
    ps = ol.crop_params(4000, 32, 40, 28, 30, "train", seed=5, file_index=1)
    oys = {p[0] for p in ps}
    oxs = {p[1] for p in ps}
    assert oys == set(range(5)) and oxs == set(range(11))
    frac = sum(p[2] for p in ps) / len(ps)
    assert 0.45 < frac < 0.55


def test_deliveries_protocol():
    # "stop" first -> nothing
    assert ol.deliveries([("stop", None)]) == []
    # m filenames deliver in order; the last loaded one waits for a
    # further message (Alg. 1) and is not delivered on a mode switch
    msgs = [("train", None), ("file", "a"), ("file", "b"), ("file", "c"), ("val", None),
            ("file", "v0"), ("file", "v1"), ("stop", None)]
    assert ol.deliveries(msgs) == [("a", "train", 0), ("b", "train", 1), ("v0", "val", 3)]
    # mode switch mid-stream re-enters the outer loop
    msgs = [("val", None), ("file", "x"), ("train", None), ("file", "y"), ("file", "z")]
    assert ol.deliveries(msgs) == [("y", "train", 1)]


def test_batch_file_format(tmp_path):
    from paper_1605_08325_b200.tm import write_batch_file
    raw, _ = _batch()
    p = str(tmp_path / "b0.pxb")
    write_batch_file(p, raw)
    assert np.array_equal(ol.read_batch_file(p), raw)
    with open(p, "r+b") as f:
        f.write(b"XXXX")
    with pytest.raises(ValueError):
        ol.read_batch_file(p)
