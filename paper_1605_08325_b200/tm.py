"""Thin ctypes binding of libtm.so (include/tm.h).  Argument marshalling only:
every step of the exchange runs in the library's sm_100a kernels.  There is no
CPU or PyTorch fallback: if libtm.so is missing or a call fails, this module
raises.

Names follow the C ABI: tm_exchange_init / tm_exchange / tm_easgd_update ...
The `Exchanger` class wraps the process-global exchanger for convenience.
"""

import ctypes
import os
import glob

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libtm.so")

TM_AR, TM_ASA, TM_ASA16, TM_EASGD = 0, 1, 2, 3
STRATEGY = {"ar": TM_AR, "asa": TM_ASA, "asa16": TM_ASA16, "easgd": TM_EASGD}
TM_OK, TM_E_ARG, TM_E_ALIGN, TM_E_STATE, TM_E_CUDA, TM_E_NCCL = 0, 1, 2, 3, 4, 5
TM_E_MISMATCH, TM_E_TIMEOUT, TM_E_NONFINITE, TM_E_OVERFLOW16 = 6, 7, 8, 9
TM_BIT_NONFINITE, TM_BIT_OVERFLOW16, TM_BIT_TIMEOUT = 1, 2, 4
TM_OP_SUM = 0x100  # SUBGD: sum instead of average
TM_PATH_AUTO, TM_PATH_STAGED, TM_PATH_DIRECT = 0, 1, 2
PATH = {"auto": TM_PATH_AUTO, "staged": TM_PATH_STAGED, "direct": TM_PATH_DIRECT}
TM_AG_SM, TM_AG_CE, TM_AG_NCCL = 0, 1, 2
ALLGATHER = {"sm": TM_AG_SM, "ce": TM_AG_CE, "nccl": TM_AG_NCCL}
TM_BLOB_BYTES = 512
TM_MAX_RANKS = 8


class TmError(RuntimeError):
    def __init__(self, code, what):
        self.code = code
        super().__init__(f"{what}: tm status {code} ({strerror(code)})")


class tm_world(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("size", ctypes.c_int32),
                ("device", ctypes.c_int32), ("nlocal", ctypes.c_int32)]


class tm_layout_info(ctypes.Structure):
    _fields_ = [("nparams", ctypes.c_int64), ("seg_len", ctypes.c_int64),
                ("chunk_len", ctypes.c_int64), ("k", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("nlocal", ctypes.c_int32), ("strategy", ctypes.c_int32),
                ("ctas_per_rank", ctypes.c_int32), ("threads", ctypes.c_int32),
                ("sm_count", ctypes.c_int32), ("wire_bytes", ctypes.c_int32),
                ("lib_bytes", ctypes.c_int64), ("epoch", ctypes.c_uint32),
                ("path", ctypes.c_int32), ("staged_kernel", ctypes.c_int32),
                ("allgather", ctypes.c_int32), ("selfcheck", ctypes.c_int32)]


_lib = None

_P = ctypes.c_void_p
_SIGS = {
    "tm_exchange_init": (ctypes.c_int, [ctypes.c_int64, ctypes.POINTER(tm_world), ctypes.c_int]),
    "tm_bootstrap_export": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_size_t)]),
    "tm_bootstrap_import": (ctypes.c_int, [_P, ctypes.c_size_t]),
    "tm_exchange": (ctypes.c_int, [_P, _P]),
    "tm_exchange_group": (ctypes.c_int, [ctypes.POINTER(_P), ctypes.c_int, _P]),
    "tm_exchange_range": (ctypes.c_int, [_P, ctypes.c_int64, ctypes.c_int64, _P]),
    "tm_bsp_step": (ctypes.c_int, [_P, _P, _P, ctypes.c_float, ctypes.c_float, ctypes.c_int, _P]),
    "tm_bsp_step_group": (ctypes.c_int, [ctypes.POINTER(_P), ctypes.POINTER(_P), ctypes.POINTER(_P),
                                         ctypes.c_int, ctypes.c_float, ctypes.c_float, ctypes.c_int, _P]),
    "tm_exchange_group_range": (ctypes.c_int, [ctypes.POINTER(_P), ctypes.c_int, ctypes.c_int64,
                                               ctypes.c_int64, _P]),
    "tm_easgd_update": (ctypes.c_int, [_P, _P, ctypes.c_float, _P]),
    "tm_easgd_update_ex": (ctypes.c_int, [_P, _P, ctypes.c_int64, ctypes.c_float, ctypes.c_int, _P]),
    "tm_easgd_round": (ctypes.c_int, [ctypes.POINTER(_P), ctypes.c_int, ctypes.POINTER(ctypes.c_int32),
                                      ctypes.c_int, _P, ctypes.c_int64, ctypes.c_float, _P]),
    "tm_easgd_center": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(_P)]),
    "tm_easgd_update_sharded": (ctypes.c_int, [_P, ctypes.c_float, ctypes.c_int, _P]),
    "tm_easgd_update_locked": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_float, _P]),
    "tm_easgd_set_order_log": (ctypes.c_int, [_P, ctypes.c_int]),
    "tm_exchange_status": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_uint32)]),
    "tm_layout": (ctypes.c_int, [ctypes.POINTER(tm_layout_info)]),
    "tm_set_timeout_ns": (ctypes.c_int, [ctypes.c_uint64]),
    "tm_set_range_ctas": (ctypes.c_int, [ctypes.c_int]),
    "tm_set_path": (ctypes.c_int, [ctypes.c_int]),
    "tm_set_allgather": (ctypes.c_int, [ctypes.c_int]),
    "tm_set_phase_log": (ctypes.c_int, [_P, ctypes.c_int64]),
    "tm_exchange_finalize": (ctypes.c_int, []),
    "tm_strerror": (ctypes.c_char_p, [ctypes.c_int]),
    "tm_cast_rn16": (ctypes.c_int, [_P, _P, ctypes.c_int64, _P]),
    "tm_loader_create": (ctypes.c_int, [_P, _P, _P]),
    "tm_loader_send": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_char_p]),
    "tm_loader_send_after": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_char_p, _P]),
    "tm_loader_wait": (ctypes.c_int, [_P, ctypes.c_int64]),
    "tm_loader_destroy": (ctypes.c_int, [_P]),
}


def _torch_nccl_path():
    try:
        import nvidia.nccl  # type: ignore
        for base in nvidia.nccl.__path__:
            hits = glob.glob(os.path.join(base, "lib", "libnccl.so*"))
            if hits:
                return sorted(hits)[0]
    except Exception:
        pass
    return ""


def lib():
    """Load libtm.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build() "
                               "(python -m paper_1605_08325_b200.build)")
        if not os.environ.get("TM_NCCL_LIB"):
            os.environ["TM_NCCL_LIB"] = _torch_nccl_path()
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def strerror(code):
    return lib().tm_strerror(int(code)).decode()


def _check(code, what):
    if code != TM_OK:
        raise TmError(code, what)


def _stream_handle(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


# What the process's exchanger was initialised with (set by tm_exchange_init,
# cleared by tm_exchange_finalize): the C ABI takes bare device pointers and
# cannot check a tensor's length or device, so the wrappers do, before a short
# tensor or one on another GPU reaches a kernel.
_ctx = {}


def _fp32_cuda(t, n=None, min_n=None):
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float32
            and t.is_contiguous()):
        raise TypeError("expected a contiguous float32 CUDA tensor")
    if n is not None and t.numel() != n:
        raise ValueError(f"expected {n} elements, got {t.numel()}")
    if min_n is not None and t.numel() < min_n:
        raise ValueError(f"expected at least {min_n} elements, got {t.numel()}")
    return ctypes.c_void_p(t.data_ptr())


def _param_buf(t):
    """A caller buffer of the exchanger: fp32[nparams] on the exchanger's device."""
    p = _fp32_cuda(t, n=_ctx.get("nparams"))
    if "device" in _ctx and t.device.index != _ctx["device"]:
        raise ValueError(f"tensor on cuda:{t.device.index}, exchanger on cuda:{_ctx['device']}")
    return p


def _check_range(offset, count):
    P = _ctx.get("nparams")
    if offset < 0 or count < 0 or (P is not None and offset + count > P):
        raise ValueError(f"range [{offset}, {offset + count}) outside [0, {P})")


# ------------------------------------------------------------------ raw calls

def tm_exchange_init(nparams, rank, size, device, nlocal, strategy):
    w = tm_world(rank, size, device, nlocal)
    _check(lib().tm_exchange_init(int(nparams), ctypes.byref(w), int(strategy)), "tm_exchange_init")
    _ctx.clear()
    _ctx.update(nparams=int(nparams), device=int(device), nlocal=int(nlocal))


def tm_bootstrap_export():
    buf = ctypes.create_string_buffer(TM_BLOB_BYTES)
    n = ctypes.c_size_t(0)
    _check(lib().tm_bootstrap_export(buf, ctypes.byref(n)), "tm_bootstrap_export")
    return buf.raw[: n.value]


def tm_bootstrap_import(blobs):
    each = len(blobs[0])
    joined = b"".join(blobs)
    _check(lib().tm_bootstrap_import(joined, each), "tm_bootstrap_import")


def tm_exchange(buf, stream=None):
    _check(lib().tm_exchange(_param_buf(buf), _stream_handle(stream)), "tm_exchange")


def tm_exchange_group(bufs, stream=None):
    arr = (ctypes.c_void_p * len(bufs))(*[_param_buf(b).value for b in bufs])
    _check(lib().tm_exchange_group(arr, len(bufs), _stream_handle(stream)), "tm_exchange_group")


def tm_exchange_range(buf, offset, count, stream=None):
    _check_range(int(offset), int(count))
    _check(lib().tm_exchange_range(_param_buf(buf), int(offset), int(count), _stream_handle(stream)),
           "tm_exchange_range")


def tm_exchange_group_range(bufs, offset, count, stream=None):
    _check_range(int(offset), int(count))
    arr = (ctypes.c_void_p * len(bufs))(*[_param_buf(b).value for b in bufs])
    _check(lib().tm_exchange_group_range(arr, len(bufs), int(offset), int(count),
                                         _stream_handle(stream)), "tm_exchange_group_range")


def tm_bsp_step(w, v, grad, lr, mu, exchange_momentum=False, stream=None):
    _check(lib().tm_bsp_step(_param_buf(w), _param_buf(v), _param_buf(grad), ctypes.c_float(lr),
                             ctypes.c_float(mu), int(bool(exchange_momentum)), _stream_handle(stream)),
           "tm_bsp_step")


def tm_bsp_step_group(ws, vs, grads, lr, mu, exchange_momentum=False, stream=None):
    n = len(ws)
    arr = lambda ts: (ctypes.c_void_p * n)(*[_param_buf(t).value for t in ts])  # noqa: E731
    _check(lib().tm_bsp_step_group(arr(ws), arr(vs), arr(grads), n, ctypes.c_float(lr),
                                   ctypes.c_float(mu), int(bool(exchange_momentum)),
                                   _stream_handle(stream)), "tm_bsp_step_group")


def tm_easgd_update(worker, center, alpha, stream=None):
    P = _ctx.get("nparams")
    cptr = center if isinstance(center, int) else _fp32_cuda(center, min_n=P).value
    _check(lib().tm_easgd_update(_param_buf(worker), _P(cptr), ctypes.c_float(alpha), _stream_handle(stream)),
           "tm_easgd_update")


def tm_easgd_update_ex(worker, center, alpha, concurrent=False, stream=None, n=None):
    wptr = _fp32_cuda(worker)
    n = worker.numel() if n is None else int(n)
    if n < 0 or n > worker.numel():
        raise ValueError(f"n = {n} outside [0, {worker.numel()}]")
    cptr = center if isinstance(center, int) else _fp32_cuda(center, min_n=n).value
    mode = 2 if concurrent == "exact" else int(concurrent)  # 0, 1 (red.add), 2 / "exact" (CAS loop)
    if isinstance(center, torch.Tensor) and center.device != worker.device:
        raise ValueError(f"centre on {center.device}, worker on {worker.device}: pass a peer-mapped "
                         "pointer (int) for a centre on another GPU")
    _check(lib().tm_easgd_update_ex(wptr, _P(cptr), int(n), ctypes.c_float(alpha),
                                    mode, _stream_handle(stream)), "tm_easgd_update_ex")


def tm_easgd_round(workers, order, center, alpha, stream=None):
    n = center.numel()
    if any(w.device != center.device for w in workers):
        raise ValueError("workers and centre must be on one device")
    arr = (ctypes.c_void_p * len(workers))(*[_fp32_cuda(w, n).value for w in workers])
    o = (ctypes.c_int32 * len(order))(*[int(i) for i in order])
    _check(lib().tm_easgd_round(arr, len(workers), o, len(order), _fp32_cuda(center), int(n),
                                ctypes.c_float(alpha), _stream_handle(stream)), "tm_easgd_round")


def tm_easgd_update_sharded(worker, alpha, concurrent=False, stream=None):
    mode = 2 if concurrent == "exact" else int(concurrent)
    _check(lib().tm_easgd_update_sharded(_param_buf(worker), ctypes.c_float(alpha),
                                         mode, _stream_handle(stream)),
           "tm_easgd_update_sharded")


def tm_easgd_update_locked(worker, worker_id, alpha, stream=None):
    _check(lib().tm_easgd_update_locked(_param_buf(worker), int(worker_id), ctypes.c_float(alpha),
                                        _stream_handle(stream)), "tm_easgd_update_locked")


TM_LOCK_CHUNK = 4096  # elements per lock of the locked EASGD mode (include/tm.h, tm_easgd_update_locked)


def tm_easgd_set_order_log(log, max_updates_per_chunk):
    """log: int32 CUDA tensor of >= k * nchunk * max entries (nchunk =
    ceil(seg_len / 4096)) on the exchanger's device, or None."""
    ptr = None
    if log is not None:
        lay = tm_layout()
        need = lay["k"] * -(-lay["seg_len"] // TM_LOCK_CHUNK) * int(max_updates_per_chunk)
        if not (isinstance(log, torch.Tensor) and log.is_cuda and log.dtype == torch.int32
                and log.is_contiguous()):
            raise TypeError("expected a contiguous int32 CUDA tensor")
        if log.numel() < need:
            raise ValueError(f"order log holds {log.numel()} entries, needs {need}")
        if "device" in _ctx and log.device.index != _ctx["device"]:
            raise ValueError(f"order log on cuda:{log.device.index}, exchanger on cuda:{_ctx['device']}")
        ptr = ctypes.c_void_p(log.data_ptr())
    _check(lib().tm_easgd_set_order_log(ptr, int(max_updates_per_chunk)), "tm_easgd_set_order_log")


def tm_easgd_center(owner_rank):
    p = ctypes.c_void_p(0)
    _check(lib().tm_easgd_center(int(owner_rank), ctypes.byref(p)), "tm_easgd_center")
    return p.value


def tm_exchange_status(stream=None):
    bits = ctypes.c_uint32(0)
    code = lib().tm_exchange_status(_stream_handle(stream), ctypes.byref(bits))
    return code, bits.value


def tm_layout():
    info = tm_layout_info()
    _check(lib().tm_layout(ctypes.byref(info)), "tm_layout")
    return {f: getattr(info, f) for f, _ in info._fields_}


def tm_set_timeout_ns(ns):
    _check(lib().tm_set_timeout_ns(int(ns)), "tm_set_timeout_ns")


def tm_set_range_ctas(ctas):
    _check(lib().tm_set_range_ctas(int(ctas)), "tm_set_range_ctas")


def tm_set_path(path):
    _check(lib().tm_set_path(PATH[path] if isinstance(path, str) else int(path)), "tm_set_path")


def tm_set_allgather(mode):
    _check(lib().tm_set_allgather(ALLGATHER[mode] if isinstance(mode, str) else int(mode)),
           "tm_set_allgather")


def tm_set_phase_log(buf):
    """buf: int64 CUDA tensor (>= nlocal*C*8 slots) or None."""
    _check(lib().tm_set_phase_log(None if buf is None else ctypes.c_void_p(buf.data_ptr()),
                                  0 if buf is None else buf.numel()), "tm_set_phase_log")


def tm_exchange_finalize():
    _ctx.clear()
    _check(lib().tm_exchange_finalize(), "tm_exchange_finalize")


def tm_cast_rn16(x, out16=None, stream=None):
    """Device binary16 RNE rounding (the exchange's own); returns int16 bit patterns."""
    if out16 is None:
        out16 = torch.empty(x.numel(), dtype=torch.int16, device=x.device)
    if not (out16.dtype in (torch.int16, torch.float16) and out16.device == x.device
            and out16.is_contiguous() and out16.numel() >= x.numel()):
        raise ValueError("out16: a contiguous 16-bit tensor of >= x.numel() elements on x's device")
    _check(lib().tm_cast_rn16(_fp32_cuda(x), _P(out16.data_ptr()), x.numel(), _stream_handle(stream)),
           "tm_cast_rn16")
    return out16


def device_view(ptr, n, device=None):
    """A float32 torch tensor aliasing n floats of library-owned device memory
    at `ptr` (e.g. tm_easgd_center's pointer).  No copy."""

    class _Iface:
        __cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f4",
                                    "data": (int(ptr), False), "version": 2}

    return torch.as_tensor(_Iface(), device=device or torch.cuda.current_device())


# ------------------------------------------------------------ parallel loading

TM_LOADER_TRAIN, TM_LOADER_VAL, TM_LOADER_STOP, TM_LOADER_FILE = 0, 1, 2, 3
TM_E_IO = 10


class tm_loader_config(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("c", ctypes.c_int32), ("h", ctypes.c_int32),
                ("w", ctypes.c_int32), ("crop_h", ctypes.c_int32), ("crop_w", ctypes.c_int32),
                ("device", ctypes.c_int32), ("seed", ctypes.c_uint64),
                ("mean", ctypes.POINTER(ctypes.c_float))]


def write_batch_file(path, raw):
    """Write a uint8 [n, c, h, w] batch as a PXB1 file."""
    import struct
    import numpy as np
    raw = np.ascontiguousarray(raw, dtype=np.uint8)
    if raw.ndim != 4:
        raise ValueError("expected [n, c, h, w]")
    with open(path, "wb") as f:
        f.write(b"PXB1" + struct.pack("<4I", *raw.shape))
        f.write(raw.tobytes())


class Loader:
    """Alg. 1's parallel loading process (tm_loader_*): a native loader thread
    that reads batch files, preprocesses them on the GPU and hands each batch to
    `input_x` when the trainer asks for the next file."""

    def __init__(self, n, c, h, w, crop_h, crop_w, mean, input_x, seed=0, device=None):
        import numpy as np
        self._mean = np.ascontiguousarray(mean, dtype=np.float32)
        if self._mean.shape != (c, h, w):
            raise ValueError("mean image must be [c, h, w]")
        _fp32_cuda(input_x, n * c * crop_h * crop_w)
        self.input_x = input_x
        cfg = tm_loader_config(n, c, h, w, crop_h, crop_w,
                               input_x.device.index if device is None else device, seed,
                               self._mean.ctypes.data_as(ctypes.POINTER(ctypes.c_float)))
        self._h = ctypes.c_void_p()
        _check(lib().tm_loader_create(ctypes.byref(cfg), ctypes.c_void_p(input_x.data_ptr()),
                                      ctypes.byref(self._h)), "tm_loader_create")

    def send(self, kind, filename=None, stream=None):
        """A FILE message's copy into input_x waits for the work enqueued so far
        on `stream` (default: the current stream), i.e. the trainer's kernels
        still reading the previous batch."""
        k = {"train": TM_LOADER_TRAIN, "val": TM_LOADER_VAL, "stop": TM_LOADER_STOP,
             "file": TM_LOADER_FILE}[kind]
        _check(lib().tm_loader_send_after(self._h, k, None if filename is None else filename.encode(),
                                          _stream_handle(stream)), "tm_loader_send_after")

    def wait(self, timeout_ms=-1):
        _check(lib().tm_loader_wait(self._h, int(timeout_ms)), "tm_loader_wait")

    def close(self):
        if self._h:
            lib().tm_loader_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


# ------------------------------------------------------------ convenience

def gather_blobs(mine, nprocs, group=None):
    """All-gather this process's bootstrap blob over torch.distributed; returns
    the nprocs blobs in process (rank) order, as tm_bootstrap_import expects."""
    import torch.distributed as dist
    if dist.get_world_size(group) != nprocs:
        raise ValueError(f"process group has {dist.get_world_size(group)} ranks, expected {nprocs}")
    blobs = [None] * nprocs
    dist.all_gather_object(blobs, bytes(mine), group=group)
    if any(len(b) != len(blobs[0]) for b in blobs):
        raise ValueError("bootstrap blobs differ in length")
    return blobs


class Exchanger:
    """Process-global exchanger.

    Single-process group (k workers on one device):
        ex = Exchanger(P, "asa16", size=k, nlocal=k); ex.exchange([b0, ..., bk-1])
    One process per GPU under torch.distributed (bootstrap over `group`):
        ex = Exchanger(P, "asa16", rank=r, size=k, device=d, nlocal=1, group=pg)
        ex.exchange(buf)
    """

    def __init__(self, nparams, strategy, rank=0, size=1, device=None, nlocal=None,
                 group=None, timeout_s=None, path="auto", op="avg", allgather=None):
        if device is None:
            device = torch.cuda.current_device()
        nlocal = size if nlocal is None else nlocal
        self.nparams, self.size, self.nlocal, self.rank = int(nparams), size, nlocal, rank
        self.strategy = strategy
        torch.cuda.set_device(device)
        if op not in ("avg", "sum"):
            raise ValueError(op)
        tm_exchange_init(nparams, rank, size, device, nlocal,
                         STRATEGY[strategy] | (TM_OP_SUM if op == "sum" else 0))
        if timeout_s is not None:
            tm_set_timeout_ns(int(timeout_s * 1e9))
        if path != "auto":
            tm_set_path(path)
        try:
            if nlocal != size:
                tm_bootstrap_import(gather_blobs(tm_bootstrap_export(), size // nlocal, group))
            if allgather is not None:
                tm_set_allgather(allgather)
        except Exception:
            tm_exchange_finalize()  # no half-initialised process-global exchanger left behind
            raise

    def exchange(self, bufs, stream=None):
        if isinstance(bufs, torch.Tensor):
            tm_exchange(bufs, stream)
        else:
            tm_exchange_group(list(bufs), stream)

    def exchange_range(self, bufs, offset, count, stream=None):
        """Exchange elements [offset, offset + count) only (one bucket)."""
        if isinstance(bufs, torch.Tensor):
            tm_exchange_range(bufs, offset, count, stream)
        else:
            tm_exchange_group_range(list(bufs), offset, count, stream)

    def bsp_step(self, w, v, grad, lr, mu, exchange_momentum=False, stream=None):
        """Momentum-SGD step of every local rank, then the exchange (fused in
        one pass for a single-process group on the direct path)."""
        if isinstance(w, torch.Tensor):
            tm_bsp_step(w, v, grad, lr, mu, exchange_momentum, stream)
        else:
            tm_bsp_step_group(list(w), list(v), list(grad), lr, mu, exchange_momentum, stream)

    def status(self, stream=None):
        return tm_exchange_status(stream)

    def layout(self):
        return tm_layout()

    def center(self, owner_rank=0):
        return tm_easgd_center(owner_rank)

    def center_shard(self, owner_rank):
        """owner_rank's centre shard as a torch tensor view (no copy)."""
        L = self.layout()["seg_len"]
        n = max(0, min(L, self.nparams - owner_rank * L))
        return device_view(tm_easgd_center(owner_rank), n)

    def finalize(self):
        tm_exchange_finalize()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.finalize()
