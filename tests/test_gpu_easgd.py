"""GPU parity of the EASGD kernels against oracle/easgd.py."""

import numpy as np
import pytest
import torch

from gpu_helpers import assert_bitwise, to_dev, to_host
from oracle.easgd import easgd_sequence, easgd_update
from paper_1605_08325_b200 import tm
from paper_1605_08325_b200.inputs import worker_buffer

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("alpha", [0.5, 0.0625, 0.3])
@pytest.mark.parametrize("dist", ["D1", "D2", "D3", "D6"])
def test_update_bitwise(alpha, dist):
    for n in (1, 3, 4, 1000, 1_000_003):
        x = worker_buffer(n, dist, 0, config=40)
        c = worker_buffer(n, dist, 1, config=40)
        xd, cd = to_dev([x, c])
        tm.tm_easgd_update_ex(xd, cd, alpha)
        gx, gc = to_host([xd, cd])
        wx, wc = easgd_update(x, c, alpha)
        assert_bitwise(gx, wx, f"x n={n}")
        assert_bitwise(gc, wc, f"c n={n}")


def test_update_unaligned_views():
    n = 100_001
    x = worker_buffer(n + 1, "D1", 0, config=41)
    c = worker_buffer(n + 3, "D1", 1, config=41)
    xd, cd = to_dev([x, c])
    tm.tm_easgd_update_ex(xd[1:], cd[3:], 0.3)  # 4- and 12-byte offsets: scalar path
    gx, gc = to_host([xd, cd])
    wx, wc = easgd_update(x[1:], c[3:], 0.3)
    assert_bitwise(gx[1:], wx)
    assert_bitwise(gc[3:], wc)
    assert gx[0] == x[0] and np.array_equal(gc[:3], c[:3])


def test_update_with_context_and_library_centre():
    n = 65_537
    with tm.Exchanger(n, "easgd", size=1, nlocal=1) as ex:
        centre = tm.device_view(ex.center(0), n)
        x = worker_buffer(n, "D2", 0, config=42)
        c0 = worker_buffer(n, "D2", 1, config=42)
        xd = to_dev([x])[0]
        centre.copy_(torch.from_numpy(c0))
        tm.tm_easgd_update(xd, centre, 0.5)
        gx, gc = to_host([xd, centre])
        wx, wc = easgd_update(x, c0, 0.5)
        assert_bitwise(gx, wx)
        assert_bitwise(gc, wc)


def test_concurrent_mode_serial_stream_equals_exclusive():
    """red.add on one stream (no contention): fl(c + e) exactly as the oracle."""
    n = 500_000
    x = worker_buffer(n, "D1", 0, config=43)
    c = worker_buffer(n, "D1", 1, config=43)
    xd, cd = to_dev([x, c])
    tm.tm_easgd_update_ex(xd, cd, 0.0625, concurrent=True)
    gx, gc = to_host([xd, cd])
    wx, wc = easgd_update(x, c, 0.0625)
    assert_bitwise(gx, wx)
    assert_bitwise(gc, wc)


@pytest.mark.parametrize("n", [1_000_003, 5_123, 1_027])
@pytest.mark.parametrize("order", [[0, 1, 2, 3, 4, 5, 6, 7], [7, 2, 5, 0, 2, 1], [3], [4, 0, 6, 1, 2]])
def test_fused_round_equals_arrival_order_sequence(order, n):
    """Distinct arrival orders run the TMA-engine round kernel (whole 1024-element
    tiles + register tail), repeated workers the generic kernel."""
    nw = 8
    W = [worker_buffer(n, "D3", r, config=44) for r in range(nw)]
    c = worker_buffer(n, "D3", 99, config=44)
    Wd = to_dev(W)
    cd = to_dev([c])[0]
    tm.tm_easgd_round(Wd, order, cd, 0.5 / 8)
    gW = to_host(Wd)
    gc = to_host([cd])[0]
    wW, wc = easgd_sequence(W, c, 0.5 / 8, order)
    assert_bitwise(gc, wc, "centre")
    for r in range(nw):
        assert_bitwise(gW[r], wW[r], f"worker {r}")


def test_concurrent_rounds_on_two_streams_bitwise():
    """Two servers' rounds (disjoint centres and workers) issued on two streams
    with no ordering between them, three times each: the dynamic-tile round
    kernel claims tiles from a per-launch counter pair (a per-device ring), so
    concurrent launches never split each other's tile claims.  Each centre and
    worker set ends bitwise at the oracle's arrival-order sequence."""
    n, nw = 3_000_017, 8
    orders = [[0, 1, 2, 3, 4, 5, 6, 7], [5, 3, 1, 7, 0, 2, 6, 4]]
    Ws = [[worker_buffer(n, "D2", 10 * s + r, config=46) for r in range(nw)] for s in range(2)]
    cs = [worker_buffer(n, "D2", 90 + s, config=46) for s in range(2)]
    Wds = [to_dev(W) for W in Ws]
    cds = [to_dev([c])[0] for c in cs]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    torch.cuda.synchronize()
    for _ in range(3):
        for s in range(2):
            tm.tm_easgd_round(Wds[s], orders[s], cds[s], 0.5 / 8, stream=streams[s])
    torch.cuda.synchronize()
    for s in range(2):
        wW, wc = Ws[s], cs[s]
        for _ in range(3):
            wW, wc = easgd_sequence(wW, wc, 0.5 / 8, orders[s])
        assert_bitwise(to_host([cds[s]])[0], wc, f"centre {s}")
        gW = to_host(Wds[s])
        for r in range(nw):
            assert_bitwise(gW[r], wW[r], f"server {s} worker {r}")


def test_concurrent_workers_invariants():
    """8 workers update one centre concurrently from 8 streams (Q15: no bitwise
    oracle).  Invariants: sum_w x_w + c conserved within the rounding bound, and
    each worker moved toward the centre it read."""
    n = 1 << 20
    nw = 8
    alpha = 0.5 / nw
    W = [worker_buffer(n, "D1", r, config=45) for r in range(nw)]
    c = worker_buffer(n, "D1", 99, config=45)
    Wd = to_dev(W)
    cd = to_dev([c])[0]
    streams = [torch.cuda.Stream() for _ in range(nw)]
    torch.cuda.synchronize()
    for w, s in zip(Wd, streams):
        tm.tm_easgd_update_ex(w, cd, alpha, concurrent=True, stream=s)
    torch.cuda.synchronize()
    gW = to_host(Wd)
    gc = to_host([cd])[0]
    tot0 = sum(w.astype(np.float64) for w in W) + c
    tot1 = sum(w.astype(np.float64) for w in gW) + gc
    scale = sum(np.abs(w.astype(np.float64)) for w in gW) + np.abs(gc)
    assert np.all(np.abs(tot1 - tot0) <= 2 * (nw + 1) * 2.0 ** -24 * scale + 1e-30)
    # the serial-order oracle's centre is within the reordering bound
    _, wc = easgd_sequence(W, c, alpha, list(range(nw)))
    assert np.max(np.abs(gc.astype(np.float64) - wc)) < 0.25


@pytest.mark.parametrize("mode", [True, "exact", "exact32"])
@pytest.mark.parametrize("scale", ["D1", "subnormal"])
@pytest.mark.parametrize("sharded", [False, True])
def test_concurrent_updates_are_admissible_interleavings(mode, scale, sharded, monkeypatch):
    """4 workers update one centre concurrently from 4 streams (PAPER L573-581,
    reading Q15).  Every sampled element of every worker and of the centre must
    equal, bit for bit, one result of the oracle's enumeration of all
    interleavings (oracle.easgd.easgd_concurrent_admissible: every order of the
    atomic adds, every centre state a worker can have read); the fast mode
    (red.add) against the flushing add, the exact mode (CAS) against the IEEE
    add.  Inputs of the 'subnormal' scale put the centre and the elastic
    differences in fp32's subnormal range, where the two modes differ.  The
    exact mode on a centre of this GPU takes one 128-bit CAS per 4 elements;
    "exact32" forces the 32-bit CAS per element (TM_EASGD_CAS128=0), the path
    a centre on a peer GPU takes."""
    from oracle.easgd import easgd_concurrent_admissible
    if mode == "exact32":
        monkeypatch.setenv("TM_EASGD_CAS128", "0")
        mode = "exact"
    nw, P = 4, 1 << 20
    alpha = np.float32(0.3)
    W = [worker_buffer(P, "D1", r, config=49) for r in range(nw)]
    c = worker_buffer(P, "D1", 98, config=49)
    if scale == "subnormal":
        f = np.float32(2.0 ** -130)
        W = [np.multiply(w, f, dtype=np.float32) for w in W]
        c = np.multiply(c, f, dtype=np.float32)
    Wd = to_dev(W)
    streams = [torch.cuda.Stream() for _ in range(nw)]
    if sharded:
        with tm.Exchanger(P, "easgd", size=nw, nlocal=nw) as ex:
            L = ex.layout()["seg_len"]
            for s in range(nw):
                sh = ex.center_shard(s)
                sh.copy_(torch.from_numpy(c[s * L: s * L + sh.numel()]))
            torch.cuda.synchronize()
            go = _hold_streams(streams)
            for w, st in zip(Wd, streams):
                tm.tm_easgd_update_sharded(w, float(alpha), concurrent=mode, stream=st)
            torch.cuda.synchronize()
            gW, gc = to_host(Wd), _read_centre(ex, P, nw)
    else:
        cd = to_dev([c])[0]
        torch.cuda.synchronize()
        go = _hold_streams(streams)
        for w, st in zip(Wd, streams):
            tm.tm_easgd_update_ex(w, cd, float(alpha), concurrent=mode, stream=st)
        torch.cuda.synchronize()
        gW, gc = to_host(Wd), to_host([cd])[0]
    del go
    idx = np.unique(np.concatenate([np.random.default_rng(5).integers(0, P, 1 << 16), np.arange(P - 64, P)]))
    ok = easgd_concurrent_admissible([w[idx] for w in W], c[idx], alpha, [g[idx] for g in gW], gc[idx],
                                     add="ftz" if mode is True else "ieee")
    bad = np.flatnonzero(~ok)
    assert bad.size == 0, (f"{bad.size} of {idx.size} sampled elements are no interleaving's result; first "
                           f"at {idx[bad[0]]}: workers {[float(g[idx[bad[0]]]) for g in gW]} centre {gc[idx[bad[0]]]}")
    # how often the updates really interleaved: elements no serial arrival order explains
    import itertools
    serial = np.zeros(idx.size, dtype=bool)
    for order in itertools.permutations(range(nw)):
        sw, sc = easgd_sequence([w[idx] for w in W], c[idx], alpha, list(order))
        if mode is True:  # the flushing add: compare through the admissibility of that one order
            continue
        m = bits_equal(sc, gc[idx])
        for a_, b_ in zip(sw, [g[idx] for g in gW]):
            m &= bits_equal(a_, b_)
        serial |= m
    if mode is not True:
        print(f"[interleaving] mode={mode} scale={scale} sharded={sharded}: "
              f"{int((~serial).sum())} of {idx.size} sampled elements match no serial arrival order")
    if scale == "subnormal" and mode is True:  # the flush is visible: the IEEE model rejects it
        ieee_ok = easgd_concurrent_admissible([w[idx] for w in W], c[idx], alpha, [g[idx] for g in gW], gc[idx],
                                              add="ieee")
        assert not ieee_ok.all()


def bits_equal(a, b):
    return np.asarray(a, np.float32).view(np.uint32) == np.asarray(b, np.float32).view(np.uint32)


def _hold_streams(streams):
    """Make the streams' next launches start together: each waits on an event
    recorded after a ~1 ms spin on the current stream, so the host enqueues every
    worker's update before any of them can run."""
    torch.cuda._sleep(2_000_000)
    go = torch.cuda.Event()
    go.record()
    for st in streams:
        st.wait_event(go)
    return go


def _sharded_setup(P, k, config):
    W = [worker_buffer(P, "D1", r, config=config) for r in range(k)]
    c0 = worker_buffer(P, "D1", 99, config=config)
    return W, c0


def _read_centre(ex, P, k):
    return np.concatenate([ex.center_shard(s).cpu().numpy() for s in range(k)])[:P]


@pytest.mark.parametrize("k,P", [(2, 1000), (4, 100_003), (8, 1_000_003), (3, 5)])
def test_sharded_centre_serial_bitwise(k, P):
    """Centre sharded by segment (rank s hosts c[s*L:(s+1)*L]); workers update
    it one at a time in arrival order -> bitwise the oracle's sequence."""
    W, c0 = _sharded_setup(P, k, 46)
    order = [(3 * t + 1) % k for t in range(k)] + [0]
    with tm.Exchanger(P, "easgd", size=k, nlocal=k) as ex:
        L = ex.layout()["seg_len"]
        for s in range(k):
            sh = ex.center_shard(s)
            if sh.numel():
                sh.copy_(torch.from_numpy(c0[s * L: s * L + sh.numel()]))
        Wd = to_dev(W)
        for w in order:
            tm.tm_easgd_update_sharded(Wd[w], 0.3)
        gW = to_host(Wd)
        gc = _read_centre(ex, P, k)
    wW, wc = easgd_sequence(W, c0, 0.3, order)
    assert_bitwise(gc, wc, "sharded centre")
    for r in range(k):
        assert_bitwise(gW[r], wW[r], f"worker {r}")


def test_sharded_centre_concurrent():
    """Concurrent mode on one stream equals the serial order; on k streams the
    invariants hold (conservation of sum_w x_w + c)."""
    k, P = 4, 262_147
    W, c0 = _sharded_setup(P, k, 47)
    alpha = 0.5 / k
    with tm.Exchanger(P, "easgd", size=k, nlocal=k) as ex:
        L = ex.layout()["seg_len"]
        for s in range(k):
            sh = ex.center_shard(s)
            sh.copy_(torch.from_numpy(c0[s * L: s * L + sh.numel()]))
        Wd = to_dev(W)
        for w in range(k):
            tm.tm_easgd_update_sharded(Wd[w], alpha, concurrent=True)
        gW, gc = to_host(Wd), _read_centre(ex, P, k)
        wW, wc = easgd_sequence(W, c0, alpha, list(range(k)))
        assert_bitwise(gc, wc)
        for r in range(k):
            assert_bitwise(gW[r], wW[r])
        # concurrent streams
        streams = [torch.cuda.Stream() for _ in range(k)]
        torch.cuda.synchronize()
        for w, s in zip(Wd, streams):
            tm.tm_easgd_update_sharded(w, alpha, concurrent=True, stream=s)
        torch.cuda.synchronize()
        gW2, gc2 = to_host(Wd), _read_centre(ex, P, k)
    tot0 = sum(w.astype(np.float64) for w in gW) + gc
    tot1 = sum(w.astype(np.float64) for w in gW2) + gc2
    scale = sum(np.abs(w.astype(np.float64)) for w in gW2) + np.abs(gc2)
    assert np.all(np.abs(tot1 - tot0) <= 2 * (k + 1) * 2.0 ** -24 * scale + 1e-30)


def test_sharded_requires_easgd_context():
    x = torch.zeros(1024, device="cuda")
    with tm.Exchanger(1024, "asa16", size=2, nlocal=2):
        with pytest.raises(tm.TmError) as e:
            tm.tm_easgd_update_sharded(x, 0.5)
        assert e.value.code == tm.TM_E_STATE


def _check_against_logged_order(W, c0, gW, gc, log, k, P, L, nw, alpha):
    """Each 4096-element chunk must equal the serial EASGD sequence in the
    arrival order the kernel logged for that chunk."""
    nch = -(-L // 4096)
    for s in range(k):
        for q in range(nch):
            lo = s * L + q * 4096
            hi = min(s * L + min(L, (q + 1) * 4096), P)
            if lo >= hi:
                continue
            order = [int(w) for w in log[(s * nch + q) * nw:(s * nch + q + 1) * nw]]
            assert sorted(order) == list(range(nw)), (s, q, order)
            ws, cc = easgd_sequence([w[lo:hi] for w in W], c0[lo:hi], alpha, order)
            assert_bitwise(gc[lo:hi], cc, f"centre chunk ({s},{q}) order {order}")
            for r in range(nw):
                assert_bitwise(gW[r][lo:hi], ws[r], f"worker {r} chunk ({s},{q})")


@pytest.mark.parametrize("k,P", [(4, 300_007), (8, 1_000_003)])
def test_locked_concurrent_updates_follow_logged_arrival_order(k, P):
    """Per-worker atomic exchange: nw workers update the sharded
    centre concurrently from nw streams; every chunk is bitwise the serial
    sequence of its logged arrival order."""
    nw = 8
    alpha = 0.5 / nw
    W = [worker_buffer(P, "D1", r, config=48) for r in range(nw)]
    c0 = worker_buffer(P, "D1", 99, config=48)
    with tm.Exchanger(P, "easgd", size=k, nlocal=k) as ex:
        L = ex.layout()["seg_len"]
        nch = -(-L // 4096)
        for s in range(k):
            sh = ex.center_shard(s)
            if sh.numel():
                sh.copy_(torch.from_numpy(c0[s * L: s * L + sh.numel()]))
        log = torch.full((k * nch * nw,), -1, dtype=torch.int32, device="cuda")
        tm.tm_easgd_set_order_log(log, nw)
        Wd = to_dev(W)
        streams = [torch.cuda.Stream() for _ in range(nw)]
        torch.cuda.synchronize()
        for r, (w, st) in enumerate(zip(Wd, streams)):
            tm.tm_easgd_update_locked(w, r, alpha, stream=st)
        torch.cuda.synchronize()
        code, _ = ex.status()
        assert code == tm.TM_OK
        gW, gc = to_host(Wd), _read_centre(ex, P, k)
        logh = log.cpu().numpy()
        tm.tm_easgd_set_order_log(None, 0)
    _check_against_logged_order(W, c0, gW, gc, logh, k, P, L, nw, alpha)


def test_fused_round_full_size_sampled():
    """Config 4 (8 workers + centre, AlexNet size, alpha = 0.5/8), the TMA-engine
    round in arrival order: sampled elements and the tail vs easgd_sequence."""
    import torch
    from paper_1605_08325_b200.inputs import WORKLOADS
    P, nw = WORKLOADS["alexnet"], 8
    order = [5, 2, 7, 0, 1, 6, 3, 4]
    W = [worker_buffer(P, "D3", r, config=45) for r in range(nw)]
    c = worker_buffer(P, "D3", 99, config=45)
    idx = np.unique(np.concatenate([np.random.default_rng(11).integers(0, P, 100_000),
                                    np.arange(P - 300, P)]))
    wW, wc = easgd_sequence([w[idx] for w in W], c[idx], 0.5 / 8, order)
    Wd = to_dev(W)
    cd = to_dev([c])[0]
    del W, c
    tm.tm_easgd_round(Wd, order, cd, 0.5 / 8)
    ti = torch.from_numpy(idx).cuda()
    assert_bitwise(cd[ti].cpu().numpy(), wc, "centre")
    for r in range(nw):
        assert_bitwise(Wd[r][ti].cpu().numpy(), wW[r], f"worker {r}")


def test_concurrent_mode_flushes_subnormals():
    """Concurrent mode adds e to the centre with the hardware float atomic
    (red.add.f32), which flushes subnormal inputs and results to signed zero (PTX
    ISA, atom/red .add.f32).  Exclusive mode keeps gradual underflow (reading Q6).
    Pinned so the documented difference stays true: elements whose e or c' is an
    fp32 subnormal differ; everything else is bitwise the exclusive update."""
    n = 4096
    x = worker_buffer(n, "D1", 0, config=46)
    c = worker_buffer(n, "D1", 1, config=46)
    x[:8] = np.float32(1e-39)  # d, e subnormal; c' = 0 + e subnormal
    c[:8] = np.float32(0.0)
    xd, cd = to_dev([x, c])
    tm.tm_easgd_update_ex(xd, cd, 0.5, concurrent=True)
    gx, gc = to_host([xd, cd])
    wx, wc = easgd_update(x, c, 0.5)
    assert_bitwise(gx, wx)  # the worker side is plain IEEE arithmetic
    assert np.all(gc[:8] == 0) and np.all(wc[:8] != 0)
    assert_bitwise(gc[8:], wc[8:])


@pytest.mark.parametrize("dist", ["D1", "D6"])
@pytest.mark.parametrize("cas128", ["1", "0"])
def test_exact_concurrent_mode_keeps_subnormals_bitwise(dist, cas128, monkeypatch):
    """Concurrent mode 2 ("exact") adds e to the centre with a compare-and-swap
    loop around one IEEE fp32 add (gradual underflow, reading Q6): a single
    worker's update is bitwise the exclusive update and the oracle's, subnormal
    e and c' included (where mode 1's float atomic flushes them).  Both CAS
    widths: 128-bit (centre on this GPU) and 32-bit (TM_EASGD_CAS128=0)."""
    monkeypatch.setenv("TM_EASGD_CAS128", cas128)
    n = 100_003
    x = worker_buffer(n, dist, 0, config=47)
    c = worker_buffer(n, dist, 1, config=47)
    x[:8] = np.float32(1e-39)
    c[:8] = np.float32(0.0)
    xd, cd = to_dev([x, c])
    tm.tm_easgd_update_ex(xd, cd, 0.5, concurrent="exact")
    gx, gc = to_host([xd, cd])
    wx, wc = easgd_update(x, c, 0.5)
    assert_bitwise(gx, wx, "worker")
    assert_bitwise(gc, wc, "centre")
    assert np.all(gc[:8] != 0)


@pytest.mark.parametrize("cas128", ["1", "0"])
def test_exact_concurrent_workers_conserve_and_keep_subnormals(cas128, monkeypatch):
    """8 workers on 8 streams in exact concurrent mode (Q15: no bitwise oracle,
    the order is the hardware's).  No update is lost: sum_w x_w + c is conserved
    within the rounding bound; and on a block of fp32-subnormal values -- where
    every subtraction, product by 2^-4 and sum is exact whatever the order (the
    values are multiples of 2^-149 below 2^-126) -- the centre is EXACTLY c plus
    the sum of the workers' moves, i.e. nothing was flushed to zero."""
    monkeypatch.setenv("TM_EASGD_CAS128", cas128)
    n = 1 << 20
    nw, alpha = 8, 0.0625
    W = [worker_buffer(n, "D1", r, config=48) for r in range(nw)]
    c = worker_buffer(n, "D1", 99, config=48)
    tiny = np.float32(2.0 ** -149)
    for w in range(nw):
        W[w][:256] = tiny * np.float32(16 * (w + 1)) * np.arange(1, 257, dtype=np.float32)
    c[:256] = np.float32(0.0)
    Wd = to_dev(W)
    cd = to_dev([c])[0]
    streams = [torch.cuda.Stream() for _ in range(nw)]
    torch.cuda.synchronize()
    for w, s in zip(Wd, streams):
        tm.tm_easgd_update_ex(w, cd, alpha, concurrent="exact", stream=s)
    torch.cuda.synchronize()
    gW = to_host(Wd)
    gc = to_host([cd])[0]
    moves = sum(W[w][:256].astype(np.float64) - gW[w][:256] for w in range(nw))
    assert np.all(gc[:256] != 0)
    assert np.array_equal(gc[:256].astype(np.float64), moves)
    tot0 = sum(w.astype(np.float64) for w in W) + c
    tot1 = sum(w.astype(np.float64) for w in gW) + gc
    scale = sum(np.abs(w.astype(np.float64)) for w in gW) + np.abs(gc)
    assert np.all(np.abs(tot1 - tot0) <= 2 * (nw + 1) * 2.0 ** -24 * scale + 1e-44)
