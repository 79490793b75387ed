"""Shared helpers for the -m gpu tests (never imported by the product path)."""

import numpy as np
import torch


def to_dev(arrs, device="cuda:0"):
    return [torch.from_numpy(np.ascontiguousarray(a)).to(device) for a in arrs]


def to_host(ts):
    torch.cuda.synchronize()
    return [t.cpu().numpy() for t in ts]


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


def assert_bitwise(got, want, msg=""):
    got = np.asarray(got, np.float32)
    want = np.asarray(want, np.float32)
    assert got.shape == want.shape, (got.shape, want.shape)
    ok = (bits(got) == bits(want)) | (np.isnan(got) & np.isnan(want))
    if not ok.all():
        i = int(np.argmax(~ok))
        raise AssertionError(f"{msg}: {int((~ok).sum())} of {ok.size} elements differ; first at {i}: "
                             f"got {got[i]!r} ({bits(got)[i]:08x}) want {want[i]!r} ({bits(want)[i]:08x})")


def q11_bound(X):
    """DESIGN.md Q11: 1e-6 * mean_j |x_ij| (fp64)."""
    return 1e-6 * np.mean(np.abs(np.stack(X).astype(np.float64)), axis=0)
