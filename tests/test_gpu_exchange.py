"""GPU parity of tm_exchange (single-process groups: k ranks on one device, the
same kernels with local pointers in the peer table) against the CPU oracle.

Bar: ASA and ASA16 bitwise; AR within Q11 (and, for the
single-process kernel whose order is ascending rank, bitwise); every rank's
result bitwise identical.
"""

import os

import numpy as np
import pytest
import torch

from gpu_helpers import assert_bitwise, q11_bound, to_dev, to_host
from oracle import exchange as ox
from paper_1605_08325_b200 import tm
from paper_1605_08325_b200.inputs import DISTS, WORKLOADS, worker_buffers

pytestmark = pytest.mark.gpu

SIZES = [1, 7, 8, 9, 255, 1024, 3001, 4099, 8195, 100003, 1_000_003]  # 3001: < one k=2 direct tile


PATHS = ["staged", "direct"]


def run_group(X, strategy, reps=1, path="auto"):
    """Exchange the k buffers X (numpy) through tm_exchange_group; returns the
    k results (numpy) and the status code."""
    k, P = len(X), X[0].shape[0]
    bufs = to_dev(X)
    with tm.Exchanger(P, strategy, size=k, nlocal=k, path=path) as ex:
        for _ in range(reps):
            ex.exchange(bufs)
        code, bits = ex.status()
        out = to_host(bufs)
    return out, code, bits


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("strategy", ["asa", "asa16"])
@pytest.mark.parametrize("k", [2, 3, 4, 5, 6, 7, 8])
def test_asa_family_bitwise_sizes(strategy, k, path):
    for P in SIZES:
        X = worker_buffers(P, k, "D1", config=1)
        out, code, _ = run_group(X, strategy, path=path)
        assert code == tm.TM_OK
        want = ox.exchange(X, strategy)
        for r in range(k):
            assert_bitwise(out[r], want[r], f"{strategy} k={k} P={P} rank {r}")


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("strategy", ["asa", "asa16"])
@pytest.mark.parametrize("dist", DISTS)
def test_asa_family_bitwise_distributions(strategy, dist, path):
    for k in (2, 8):
        X = worker_buffers(100003, k, dist, config=1)
        out, code, _ = run_group(X, strategy, path=path)
        assert code == tm.TM_OK
        want = ox.exchange(X, strategy)
        for r in range(k):
            assert_bitwise(out[r], want[r], f"{strategy} {dist} k={k} rank {r}")


@pytest.mark.parametrize("k", [2, 4, 8])
def test_ar_single_process(k):
    for dist in ("D1", "D2", "D4", "D6"):
        for P in (1, 9, 100003):
            X = worker_buffers(P, k, dist, config=2)
            out, code, _ = run_group(X, "ar")
            assert code == tm.TM_OK
            want = ox.ar_average(X)
            bound = q11_bound(X)
            for r in range(k):
                assert np.all(np.abs(out[r].astype(np.float64) - want[r]) <= bound)
                assert_bitwise(out[r], want[r], f"ar {dist} k={k} P={P}")  # ascending-rank kernel


@pytest.mark.parametrize("path", PATHS)
def test_ar_equals_asa_on_dyadics(path):
    from paper_1605_08325_b200.inputs import dyadic_buffers
    X = dyadic_buffers(65537, 8)
    a, _, _ = run_group(X, "ar")
    b, _, _ = run_group(X, "asa", path=path)
    mean = (np.sum(np.stack(X).astype(np.float64), axis=0) / 8).astype(np.float32)
    assert_bitwise(a[3], mean)
    assert_bitwise(b[5], mean)


def test_repeated_exchanges_fresh_inputs():
    """Back-to-back exchanges reuse the staging across epochs (a7)."""
    k, P = 4, 300007
    with tm.Exchanger(P, "asa16", size=k, nlocal=k, path="staged") as ex:
        for it in range(4):
            X = worker_buffers(P, k, DISTS[it], config=30 + it)
            bufs = to_dev(X)
            ex.exchange(bufs)
            ex.exchange(bufs)  # exchanging the average again: idempotent for ASA16
            out = to_host(bufs)
            want = ox.asa16_average(ox.asa16_average(X))
            for r in range(k):
                assert_bitwise(out[r], want[r], f"iter {it}")
        assert ex.layout()["epoch"] == 8


@pytest.mark.parametrize("path", PATHS)
def test_cross_rank_identity_and_status_clean(path):
    X = worker_buffers(1_000_003, 8, "D2", config=3)
    for strategy in ("asa", "asa16", "ar"):
        out, code, bits = run_group(X, strategy, path=path)
        assert code == tm.TM_OK and bits == 0
        for r in range(1, 8):
            assert_bitwise(out[r], out[0], strategy)


def test_k1_identity():
    X = worker_buffers(1001, 1, "D6")
    for strategy in ("ar", "asa", "asa16"):
        out, code, _ = run_group(X, strategy)
        assert code == tm.TM_OK
        assert_bitwise(out[0], X[0])


@pytest.mark.parametrize("path", PATHS)
def test_status_nonfinite_and_overflow(path):
    k, P = 2, 4099
    X = worker_buffers(P, k, "D1", config=4)
    X[0][10] = np.float32(np.inf)
    X[1][20] = np.float32(70000.0)
    X[1][P - 1] = np.float32(-65520.0)  # scalar tail element of the direct path
    out, code, bits = run_group(X, "asa16", path=path)
    assert bits == tm.TM_BIT_NONFINITE | tm.TM_BIT_OVERFLOW16
    assert code == tm.TM_E_OVERFLOW16
    assert np.isinf(out[0][10]) and np.isinf(out[1][20])  # IEEE: inf propagates
    ok = np.ones(P, bool)
    ok[[10, 20, P - 1]] = False
    assert np.isinf(out[0][P - 1])
    want = ox.asa16_average(X)
    assert_bitwise(out[0][ok], want[0][ok])
    X = worker_buffers(P, k, "D1", config=4)
    X[1][5] = np.float32(np.nan)
    _, code, bits = run_group(X, "asa", path=path)
    assert code == tm.TM_E_NONFINITE and bits == tm.TM_BIT_NONFINITE


def test_argument_errors():
    P = 1024
    with tm.Exchanger(P, "asa16", size=2, nlocal=2):
        a = torch.zeros(P + 1, device="cuda")
        b = torch.zeros(P, device="cuda")
        with pytest.raises(tm.TmError) as e:
            tm.tm_exchange_group([a[1:], b])  # 4-byte offset: misaligned
        assert e.value.code == tm.TM_E_ALIGN
        with pytest.raises(tm.TmError) as e:
            tm.tm_exchange_group([b])  # wrong count
        assert e.value.code == tm.TM_E_ARG
        with pytest.raises(tm.TmError) as e:
            tm.tm_exchange(b)  # nlocal != 1
        assert e.value.code == tm.TM_E_STATE
        with pytest.raises(tm.TmError) as e:
            tm.tm_exchange_init(P, 0, 2, 0, 2, tm.TM_ASA)  # already initialised
        assert e.value.code == tm.TM_E_STATE
        with pytest.raises(tm.TmError) as e:
            tm.tm_set_path(7)
        assert e.value.code == tm.TM_E_ARG
        assert tm.tm_layout()["path"] == tm.TM_PATH_DIRECT  # auto, single process
    with pytest.raises(tm.TmError):
        tm.tm_exchange_init(0, 0, 2, 0, 2, tm.TM_ASA)
    with pytest.raises(tm.TmError):
        tm.tm_exchange_init(10, 0, 9, 0, 9, tm.TM_ASA)


def test_layout_segments():
    """Segment layout a1: L = roundup(ceil(P/k), 256); chunk multiple of 256."""
    for P, k in ((60_965_224, 8), (6_998_552, 4), (1_000_003, 2), (1, 8)):
        with tm.Exchanger(P, "asa16", size=k, nlocal=k) as ex:
            lay = ex.layout()
            L = -(-(-(-P // k)) // 256) * 256
            assert lay["seg_len"] == L
            assert lay["chunk_len"] % 256 == 0
            assert lay["ctas_per_rank"] * lay["chunk_len"] >= L
            assert lay["wire_bytes"] == 2


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("P", [WORKLOADS["googlenet"], WORKLOADS["alexnet"]])
def test_full_size_sampled(P, path):
    """BASELINE sizes in the bench's launch configuration (k=8 group): sampled
    elements against the oracle's per-element definition, plus the tail."""
    k = 8
    g = np.random.default_rng(5)
    for strategy, dist in (("asa16", "D2"), ("asa", "D1")):
        X = worker_buffers(P, k, dist, config=3)
        bufs = to_dev(X)
        with tm.Exchanger(P, strategy, size=k, nlocal=k, path=path) as ex:
            ex.exchange(bufs)
            code, _ = ex.status()
        assert code == tm.TM_OK
        idx = np.unique(np.concatenate([g.integers(0, P, 200_000), np.arange(P - 300, P)]))
        vals = np.stack([x[idx] for x in X])
        want = ox.element_average(vals, strategy)
        ti = torch.from_numpy(idx).cuda()
        for r in (0, 3, 7):
            got = bufs[r][ti].cpu().numpy()
            assert_bitwise(got, want, f"{strategy} P={P} rank {r}")
        del bufs
        torch.cuda.empty_cache()


def test_device_rn16_exhaustive():
    """The device rounding (cvt.rn.f16.f32) on all 2^32 fp32 patterns against
    numpy's binary16 conversion, which the opt-in CPU test pins to the oracle's
    integer emulation on all 2^32 inputs; plus the oracle itself on a dense
    stratified subset.  NaN payloads are outside the contract (Q8)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle.fp16 import rn16
    step = 1 << 28
    nthr = max(1, min(16, os.cpu_count() or 1))

    def check_slice(xn, h, lo, hi):  # numpy releases the GIL in astype / compares
        xs, hs = xn[lo:hi], h[lo:hi]
        with np.errstate(over="ignore"):
            ref = xs.astype(np.float16).view(np.uint16)
        nan = np.isnan(xs)
        ok = np.array_equal(hs[~nan], ref[~nan])
        return ok and bool(np.all((hs[nan] & 0x7C00) == 0x7C00) and np.all((hs[nan] & 0x3FF) != 0))

    with ThreadPoolExecutor(nthr) as pool:
        for start in range(0, 1 << 32, step):
            b = torch.arange(start, start + step, dtype=torch.int64, device="cuda").to(torch.int32)
            x = b.view(torch.float32)
            h = tm.tm_cast_rn16(x).cpu().numpy().view(np.uint16)
            xn = x.cpu().numpy()
            part = step // nthr
            futs = [pool.submit(check_slice, xn, h, i * part, step if i == nthr - 1 else (i + 1) * part)
                    for i in range(nthr)]
            assert all(f.result() for f in futs), start
            sub = slice(None, None, 4099)
            nan = np.isnan(xn[sub])
            assert np.array_equal(h[sub][~nan], rn16(xn[sub])[~nan]), start


@pytest.mark.parametrize("strategy", ["asa16", "asa", "ar"])
@pytest.mark.parametrize("path", PATHS)
def test_cuda_graph_capture_and_replay(strategy, path):
    """The exchange captured once in a CUDA graph and replayed on fresh inputs
    (the staged kernel keeps its epochs on the device, so its launch parameters
    are constant)."""
    k, P = 4, 300_007
    bufs = to_dev(worker_buffers(P, k, "D2", config=60))
    with tm.Exchanger(P, strategy, size=k, nlocal=k, path=path) as ex:
        ex.exchange(bufs)  # warm-up outside capture
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            ex.exchange(bufs)
        for it in range(3):
            X = worker_buffers(P, k, DISTS[it], config=61 + it)
            for b, x in zip(bufs, X):
                b.copy_(torch.from_numpy(x))
            g.replay()
            out = to_host(bufs)
            want = ox.exchange(X, strategy)
            for r in range(k):
                assert_bitwise(out[r], want[r], f"{strategy} {path} replay {it} rank {r}")
        code, _ = ex.status()
        assert code == tm.TM_OK


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("strategy", ["asa", "asa16", "ar"])
def test_subgd_sum_mode(strategy, path):
    """TM_OP_SUM (SUBGD): the rank-order sum, no 1/k."""
    for k in (2, 3, 8):
        for P in (7, 4099, 100_003):
            X = worker_buffers(P, k, "D2", config=80)
            bufs = to_dev(X)
            with tm.Exchanger(P, strategy, size=k, nlocal=k, path=path, op="sum") as ex:
                ex.exchange(bufs)
                code, _ = ex.status()
                assert ex.layout()["strategy"] & tm.TM_OP_SUM
            assert code == tm.TM_OK
            out = to_host(bufs)
            want = ox.exchange(X, strategy, op="sum")
            for r in range(k):
                assert_bitwise(out[r], want[r], f"sum {strategy} {path} k={k} P={P} rank {r}")


@pytest.mark.parametrize("path", PATHS)
def test_subgd_sum_overflows_binary16(path):
    """A sum (unlike an average) can leave the binary16 range: 40000 + 40000 ->
    +inf on the wire, TM_E_OVERFLOW16 reported."""
    P = 4099
    X = [np.full(P, 1.0, np.float32), np.full(P, 1.0, np.float32)]
    X[0][123] = X[1][123] = np.float32(40000.0)
    X[0][P - 1] = X[1][P - 1] = np.float32(-40000.0)  # scalar tail of the direct path
    bufs = to_dev(X)
    with tm.Exchanger(P, "asa16", size=2, nlocal=2, path=path, op="sum") as ex:
        ex.exchange(bufs)
        code, bits = ex.status()
    assert code == tm.TM_E_OVERFLOW16 and bits == tm.TM_BIT_OVERFLOW16
    out = to_host(bufs)
    assert np.isposinf(out[0][123]) and np.isneginf(out[1][P - 1]) and out[0][5] == 2.0


# AlexNet per-layer (W + b) parameter counts (PAPER Table 3 total 60,965,224;
# SURVEY Appendix A1), scaled by 1/32 and rounded to multiples of 4.
ALEXNET_LAYERS = [34_944, 307_456, 885_120, 663_936, 442_624, 37_752_832, 16_781_312, 4_097_000]
SCALED_LAYERS = [max(4, (n // 32) // 4 * 4) for n in ALEXNET_LAYERS]


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("strategy", ["asa16", "asa", "ar"])
def test_bucketed_range_exchange_equals_full(strategy, path):
    """Per-layer buckets exchanged in backward order (fc8 first) with
    tm_exchange_group_range give exactly the full exchange (elementwise method);
    elements outside a bucket are untouched by it."""
    k = 4
    P = sum(SCALED_LAYERS) + 3  # + a ragged tail bucket
    sizes = SCALED_LAYERS + [3]
    offs = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
    X = worker_buffers(P, k, "D2", config=90)
    bufs = to_dev(X)
    with tm.Exchanger(P, strategy, size=k, nlocal=k, path=path) as ex:
        # first bucket alone: the rest of the buffer must be unchanged
        ex.exchange_range(bufs, int(offs[-2]), sizes[-2])
        part = to_host(bufs)
        untouched = np.ones(P, bool)
        untouched[offs[-2]: offs[-2] + sizes[-2]] = False
        for r in range(k):
            assert_bitwise(part[r][untouched], X[r][untouched], "outside the bucket")
        for off, n in list(zip(offs, sizes))[::-1][2:]:
            ex.exchange_range(bufs, int(off), int(n))
        ex.exchange_range(bufs, int(offs[-1]), sizes[-1])
        code, _ = ex.status()
    assert code == tm.TM_OK
    out = to_host(bufs)
    want = ox.exchange(X, strategy)
    for r in range(k):
        assert_bitwise(out[r], want[r], f"bucketed {strategy} {path} rank {r}")


def test_range_argument_errors():
    P = 4096
    with tm.Exchanger(P, "asa16", size=2, nlocal=2):
        b = [torch.zeros(P, device="cuda") for _ in range(2)]
        with pytest.raises(tm.TmError) as e:
            tm.tm_exchange_group_range(b, 2, 100)  # offset not a multiple of 4
        assert e.value.code == tm.TM_E_ALIGN
        with pytest.raises(ValueError):  # past nparams: the binding refuses it ...
            tm.tm_exchange_group_range(b, 4000, 100)
        import ctypes  # ... and so does the C ABI itself
        arr = (ctypes.c_void_p * 2)(*[t.data_ptr() for t in b])
        code = tm.lib().tm_exchange_group_range(arr, 2, 4000, 100,
                                                ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        assert code == tm.TM_E_ARG
        tm.tm_exchange_group_range(b, 0, 0)  # empty range: no-op


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("k,P", [(2, (1 << 31) + 4099), (8, (1 << 29) + 77)])
def test_maximum_sizes_sampled(k, P, path):
    """Buffers past 2^31 elements (8.6 GB per rank): 64-bit indexing everywhere.
    Inputs are drawn on the device (timing-free); sampled outputs, the region
    around element 2^31 and the ragged tail are checked against the oracle's
    per-element definition."""
    torch.cuda.empty_cache()
    gen = torch.Generator(device="cuda").manual_seed(2026)
    bufs = [(torch.randn(P, device="cuda", generator=gen) * 0.01) for _ in range(k)]
    g = np.random.default_rng(9)
    idx = np.unique(np.concatenate([g.integers(0, P, 100_000), np.arange(P - 1000, P),
                                    np.arange(max(0, (1 << 31) - 300), min(P, (1 << 31) + 300)),
                                    np.arange(0, 1000)]))
    ti = torch.from_numpy(idx).cuda()
    vals = np.stack([b[ti].cpu().numpy() for b in bufs])
    with tm.Exchanger(P, "asa16", size=k, nlocal=k, path=path) as ex:
        ex.exchange(bufs)
        code, _ = ex.status()
    assert code == tm.TM_OK
    want = ox.element_average(vals, "asa16")
    for r in (0, k - 1):
        assert_bitwise(bufs[r][ti].cpu().numpy(), want, f"P={P} k={k} {path} rank {r}")
    del bufs
    torch.cuda.empty_cache()


@pytest.mark.parametrize("path", PATHS)
def test_phase_log_does_not_change_results(path):
    """The diagnostic phase log (tm_set_phase_log) is monotone per CTA and leaves
    the exchange bitwise unchanged."""
    k, P = 4, 300_007
    X = worker_buffers(P, k, "D2", config=95)
    bufs = to_dev(X)
    with tm.Exchanger(P, "asa16", size=k, nlocal=k, path=path) as ex:
        C = ex.layout()["ctas_per_rank"]
        log = torch.zeros(k * C * 8, dtype=torch.int64, device="cuda")
        tm.tm_set_phase_log(log)
        ex.exchange(bufs)
        tm.tm_set_phase_log(None)
        out = to_host(bufs)
    want = ox.asa16_average(X)
    for r in range(k):
        assert_bitwise(out[r], want[r])
    st = log.cpu().numpy().reshape(-1, 8)[:, :6]
    if path == "staged":
        assert np.all(st[:, 0] > 0) and np.all(np.diff(st[:, [0, 1, 2, 3, 4, 5]], axis=1) >= 0)


def test_default_staged_flavour_by_segment_length(monkeypatch):
    """Without TM_STAGED_KERNEL: the LL kernel for segments of <= 512 Ki
    elements at k = 2, 64 Ki at k <= 4 and 8 Ki above; the two-shot LL2 kernel
    up to 1 Mi, 256 Ki and 64 Ki (which covers the one-shot's and the register
    two-phase kernel's former ranges); the TMA-engine kernel above that in a
    single-process group."""
    monkeypatch.delenv("TM_STAGED_KERNEL", raising=False)
    monkeypatch.delenv("TM_ONESHOT_MAX_L", raising=False)
    monkeypatch.delenv("TM_LL_MAX_L", raising=False)
    monkeypatch.delenv("TM_LL2_MAX_L", raising=False)
    for P, k, want in ((100_003, 2, 5), (1_048_576, 2, 5), (1_048_577 + 511, 2, 6), (2_097_152, 2, 6),
                       (2_097_153 + 511, 2, 1), (65_536 * 4, 4, 5), (65_537 * 4, 4, 6), (262_144 * 4, 4, 6),
                       (262_145 * 4, 4, 1), (8_192 * 8, 8, 5), (8_193 * 8, 8, 6), (65_536 * 8, 8, 6),
                       (65_537 * 8, 8, 1), (131_072 * 8, 8, 1), (10_000, 3, 5)):
        with tm.Exchanger(P, "asa16", size=k, nlocal=k, path="staged") as ex:
            assert ex.layout()["staged_kernel"] == want, (P, k)


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("strategy", ["asa", "asa16"])
def test_random_bit_patterns(path, strategy):
    """Uniformly random finite fp32 bit patterns (every exponent: fp32
    subnormals, values far beyond the binary16 range, huge magnitudes whose sums
    overflow to inf): bitwise against the oracle, NaN where the oracle has NaN
    (inf - inf; payloads are outside the contract, Q8).  Status reports the
    non-finite / overflow conditions."""
    g = np.random.default_rng(1605)
    for k in (2, 3, 8):
        P = 50_003
        X = []
        for _ in range(k):
            u = g.integers(0, 2 ** 32, P, dtype=np.uint64).astype(np.uint32)
            u[(u & 0x7F800000) == 0x7F800000] &= 0xBF7FFFFF  # finite inputs only
            X.append(u.view(np.float32))
        bufs = to_dev(X)
        with tm.Exchanger(P, strategy, size=k, nlocal=k, path=path) as ex:
            ex.exchange(bufs)
            code, bits_ = ex.status()
        with np.errstate(over="ignore", invalid="ignore"):
            want = ox.exchange(X, strategy)
        got = to_host(bufs)
        for r in range(k):
            assert_bitwise(got[r], want[r], f"{strategy} {path} k={k} rank {r}")
        if strategy == "asa16":
            assert bits_ & tm.TM_BIT_OVERFLOW16


def test_binding_rejects_short_buffers_and_bad_ranges():
    """The C ABI takes bare pointers; the binding checks every caller buffer's
    length against nparams and a range against [0, nparams) before any launch
    (a short tensor would otherwise be read / written out of bounds)."""
    import pytest as _pt
    P, k = 10_000, 2
    bufs = [torch.zeros(P, device="cuda") for _ in range(k)]
    with tm.Exchanger(P, "asa16", size=k, nlocal=k) as ex:
        with _pt.raises(ValueError):
            ex.exchange([bufs[0], bufs[1][:-4]])
        with _pt.raises(ValueError):
            ex.exchange_range(bufs, P - 8, 16)
        with _pt.raises(ValueError):
            ex.exchange_range(bufs, -4, 8)
        with _pt.raises(ValueError):
            ex.bsp_step(bufs, bufs, [bufs[0], bufs[1][:100]], 0.1, 0.9)
        ex.exchange(bufs)  # still usable
        assert ex.status()[0] == tm.TM_OK


def test_binding_rejects_short_order_log_and_rn16_output():
    """The order log and the rn16 output are caller device buffers the kernels
    write through bare pointers: the binding checks their size, type and device."""
    import pytest as _pt
    P, k = 3 * 4096 * 2 + 5, 2
    with tm.Exchanger(P, "easgd", size=k, nlocal=k) as ex:
        L = ex.layout()["seg_len"]
        need = k * -(-L // 4096) * 3
        with _pt.raises(ValueError):
            tm.tm_easgd_set_order_log(torch.zeros(need - 1, dtype=torch.int32, device="cuda"), 3)
        with _pt.raises(TypeError):
            tm.tm_easgd_set_order_log(torch.zeros(need, dtype=torch.float32, device="cuda"), 3)
        tm.tm_easgd_set_order_log(torch.zeros(need, dtype=torch.int32, device="cuda"), 3)
        tm.tm_easgd_set_order_log(None, 0)
    x = torch.zeros(1000, device="cuda")
    with _pt.raises(ValueError):
        tm.tm_cast_rn16(x, torch.zeros(999, dtype=torch.int16, device="cuda"))
    with _pt.raises(ValueError):
        tm.tm_cast_rn16(x, torch.zeros(1000, dtype=torch.int32, device="cuda"))


def test_failed_bootstrap_leaves_no_exchanger(monkeypatch):
    """An Exchanger whose bootstrap fails finalizes the process-global exchanger,
    so the next init succeeds (no half-initialised state left behind)."""
    import pytest as _pt

    def boom(*a, **kw):
        raise RuntimeError("bootstrap failed")
    monkeypatch.setattr(tm, "gather_blobs", boom)
    with _pt.raises(RuntimeError):
        tm.Exchanger(4096, "asa16", rank=0, size=2, nlocal=1)
    monkeypatch.undo()
    with tm.Exchanger(4096, "asa16", size=2, nlocal=2) as ex:
        assert ex.layout()["k"] == 2


@pytest.mark.parametrize("strategy", ["asa16", "asa"])
@pytest.mark.parametrize("k", [2, 3, 8])
def test_oneshot_interleaved_ranges_bitwise(monkeypatch, strategy, k):
    """The one-shot kernel double-buffers its staging by call parity (a per-rank
    device call counter): full exchanges and ranges of different layouts
    (different L' and C') interleaved, each on fresh perturbations, must all
    match the oracle bitwise -- an odd number of calls between two full
    exchanges flips the parity under a different layout."""
    monkeypatch.setenv("TM_STAGED_KERNEL", "oneshot")
    P = 12_289 * k
    X = worker_buffers(P, k, "D2", config=150)
    bufs = to_dev(X)
    plan = [(0, P), (4, 3000), (0, P), (P // 2 // 4 * 4, P - P // 2 // 4 * 4), (8, 5), (0, P)]
    with tm.Exchanger(P, strategy, size=k, nlocal=k, path="staged") as ex:
        assert ex.layout()["staged_kernel"] == 4
        want = [x.copy() for x in X]
        for i, (off, cnt) in enumerate(plan):
            d = worker_buffers(P, k, "D1", config=151 + i)
            for r in range(k):
                bufs[r].add_(torch.from_numpy(d[r]).cuda() * 1e-3)
                want[r] = np.add(want[r], np.multiply(d[r], np.float32(1e-3), dtype=np.float32), dtype=np.float32)
            if cnt == P:
                ex.exchange(bufs)
            else:
                ex.exchange_range(bufs, off, cnt)
            seg = ox.exchange([w[off:off + cnt] for w in want], strategy)
            for r in range(k):
                want[r][off:off + cnt] = seg[r]
        code, _ = ex.status()
    assert code == tm.TM_OK
    got = to_host(bufs)
    for r in range(k):
        assert_bitwise(got[r], want[r], f"rank {r}")


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("budget", [1, 8])
def test_range_cta_budget_bitwise(path, budget):
    """tm_set_range_ctas: bucket exchanges on at most `budget` CTAs per rank
    (the register direct kernel / fewer staged CTAs) give the oracle's bits."""
    k, P = 4, 300_007
    X = worker_buffers(P, k, "D2", config=160)
    bufs = to_dev(X)
    with tm.Exchanger(P, "asa16", size=k, nlocal=k, path=path) as ex:
        tm.tm_set_range_ctas(budget)
        b1, b2 = P // 3 // 4 * 4, 2 * P // 3 // 4 * 4
        for off, cnt in ((b2, P - b2), (b1, b2 - b1), (0, b1)):
            ex.exchange_range(bufs, off, cnt)
        code, _ = ex.status()
    assert code == tm.TM_OK
    want = ox.asa16_average(X)
    got = to_host(bufs)
    for r in range(k):
        assert_bitwise(got[r], want[r], f"rank {r}")


@pytest.mark.parametrize("budget", [3, 40])
def test_range_cta_budget_tma_kernel_bitwise(budget, monkeypatch):
    """TM_RANGE_TMA=1 (the A/B knob, default off): budgeted buckets of the direct
    path on the TMA kernel with a persistent grid of `budget` CTAs (buckets large
    enough for it: k * count > 8 Mi elements) and the register kernel for the
    small one -- the oracle's bits either way."""
    monkeypatch.setenv("TM_RANGE_TMA", "1")
    k, P = 4, 6_000_011
    X = worker_buffers(P, k, "D2", config=161)
    bufs = to_dev(X)
    with tm.Exchanger(P, "asa16", size=k, nlocal=k, path="direct") as ex:
        tm.tm_set_range_ctas(budget)
        b1, b2 = 100_000, P // 2 // 4 * 4
        for off, cnt in ((b2, P - b2), (b1, b2 - b1), (0, b1)):
            ex.exchange_range(bufs, off, cnt)
        code, _ = ex.status()
    assert code == tm.TM_OK
    want = ox.asa16_average(X)
    got = to_host(bufs)
    for r in range(k):
        assert_bitwise(got[r], want[r], f"rank {r}")
