"""ctypes binding of libmatchb200.so (include/matchb200.h) -- the GPU engine.

This is the Python side of the drop-in boundary: the reference's
``compile_X(p) -> run(hay)`` closures (pkg/src/matchbench/comparison.py,
bitparallel.py, automata.py) and ``brute_force_search`` (core.py:139-161)
are served by plans and searches on this engine.  PyTorch is used only for
device memory and streams.  There is no CPU fallback: if the CUDA library is
missing or no GPU is present every search raises.
"""
from __future__ import annotations

import ctypes
import os
import threading
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# MB_ENGINE_LIB selects another build of the same ABI (the bounds-checked
# libmatchb200_dbg.so in tests/test_gpu_bounds.py); default: the product library.
LIB_PATH = os.environ.get("MB_ENGINE_LIB") or os.path.join(_HERE, "libmatchb200.so")

MB_OK, MB_EINVAL, MB_ENOMEM, MB_ECUDA, MB_EOVERFLOW = 0, 1, 2, 3, 4
MB_MAX_M = 8192
FAMILIES = {"auto": 0, "swar": 1, "win4": 2, "aligned": 3, "shiftor": 4, "sampled": 5, "gram": 6}
FAMILY_NAMES = {v: k for k, v in FAMILIES.items()}

# every symbol include/matchb200.h declares
EXPORTS = (
    "mb_plan_create", "mb_plan_destroy", "mb_plan_info", "mb_plan_horspool", "mb_plan_sunday",
    "mb_plan_fwd_masks", "mb_plan_kmp", "mb_plan_gram_hash", "mb_ctx_create", "mb_ctx_destroy",
    "mb_find", "mb_find_batch", "mb_search_host", "mb_search_batch_host", "mb_histogram",
    "mb_launch_count", "mb_last_error", "mb_version", "mb_ctx_mp_batches", "mb_batch_create", "mb_batch_destroy",
    "mb_find_batch_prepared",
)


class EngineError(RuntimeError):
    pass


class _PlanOpts(ctypes.Structure):
    _fields_ = [("family", ctypes.c_int), ("sigma_hint", ctypes.c_int),
                ("hist", ctypes.POINTER(ctypes.c_int64)), ("anchor_words", ctypes.c_int)]


class _PlanInfo(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int64), ("family", ctypes.c_int), ("anchor", ctypes.c_int),
                ("delta", ctypes.c_int), ("period", ctypes.c_int), ("periodic", ctypes.c_int),
                ("stride", ctypes.c_int), ("gram", ctypes.c_int), ("words", ctypes.c_int)]


_lib = None
_lib_lock = threading.Lock()


def load_library():
    """Load libmatchb200.so (built by __graft_entry__.build()); raise if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise EngineError(
                f"CUDA engine library missing: {LIB_PATH} (run `python -c \"import __graft_entry__ as g; g.build()\"`)"
            )
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        P64 = ctypes.POINTER(ctypes.c_int64)
        L.mb_plan_create.argtypes = [vp, i64, ctypes.POINTER(_PlanOpts), ctypes.POINTER(vp)]
        L.mb_plan_create.restype = i32
        L.mb_plan_destroy.argtypes = [vp]
        L.mb_plan_destroy.restype = None
        L.mb_plan_info.argtypes = [vp, ctypes.POINTER(_PlanInfo)]
        L.mb_plan_info.restype = i32
        for fn in ("mb_plan_horspool", "mb_plan_sunday", "mb_plan_kmp"):
            getattr(L, fn).argtypes = [vp, vp]
            getattr(L, fn).restype = i32
        L.mb_plan_fwd_masks.argtypes = [vp, vp, i64]
        L.mb_plan_fwd_masks.restype = i32
        L.mb_plan_gram_hash.argtypes = [vp, i32, vp]
        L.mb_plan_gram_hash.restype = i32
        L.mb_ctx_create.argtypes = [i32, ctypes.POINTER(vp)]
        L.mb_ctx_create.restype = i32
        L.mb_ctx_destroy.argtypes = [vp]
        L.mb_ctx_destroy.restype = None
        L.mb_find.argtypes = [vp, vp, vp, i64, vp, i64, vp, vp]
        L.mb_find.restype = i32
        L.mb_find_batch.argtypes = [vp, vp, i32, vp, i64, vp, i64, vp, vp]
        L.mb_find_batch.restype = i32
        L.mb_search_host.argtypes = [vp, vp, i64, vp, i64, vp, i64, P64]
        L.mb_search_host.restype = i32
        L.mb_search_batch_host.argtypes = [vp, vp, vp, i32, vp, i64, vp, i64, vp]
        L.mb_search_batch_host.restype = i32
        L.mb_histogram.argtypes = [vp, vp, i64, vp, vp]
        L.mb_histogram.restype = i32
        L.mb_batch_create.argtypes = [vp, i32, ctypes.POINTER(vp)]
        L.mb_batch_create.restype = i32
        L.mb_batch_destroy.argtypes = [vp]
        L.mb_batch_destroy.restype = None
        L.mb_find_batch_prepared.argtypes = [vp, vp, vp, i64, vp, i64, vp, vp]
        L.mb_find_batch_prepared.restype = i32
        L.mb_ctx_mp_batches.argtypes = [vp]
        L.mb_ctx_mp_batches.restype = i64
        L.mb_launch_count.argtypes = []
        L.mb_launch_count.restype = i64
        L.mb_last_error.argtypes = []
        L.mb_last_error.restype = ctypes.c_char_p
        L.mb_version.argtypes = []
        L.mb_version.restype = ctypes.c_char_p
        _lib = L
        return L


def _check(rc: int):
    if rc == MB_OK:
        return
    msg = load_library().mb_last_error().decode(errors="replace")
    if rc == MB_EINVAL:
        raise ValueError(msg)
    if rc == MB_ENOMEM:
        raise MemoryError(msg)
    raise EngineError(f"matchb200 error {rc}: {msg}")


def mp_batches() -> int:
    """Batched searches of this thread's context that took the K5 multi-pattern pass."""
    return int(load_library().mb_ctx_mp_batches(context().handle))


def launch_count() -> int:
    """How many of this library's kernels have been launched in this process."""
    return int(load_library().mb_launch_count())


@dataclass(frozen=True)
class PlanInfo:
    m: int
    family: str
    anchor: int
    delta: int
    period: int
    periodic: bool
    stride: int = 0  # K3 / K1G sampling stride (bytes)
    gram: int = 0    # K3 / K1G gram length (bytes)
    words: int = 0   # ALIGNED anchor words (window 4 * words + 3 bytes)


class Plan:
    """Immutable compiled pattern (the compile_X(p) analogue).  Shareable
    across threads; owns a device copy of the pattern and its scan params."""

    __slots__ = ("_h", "pattern", "m", "__weakref__")

    def __init__(self, pattern: bytes, family: str = "auto", hist=None, anchor_words: int = 0):
        L = load_library()
        p = bytes(pattern)
        if not p:
            raise ValueError("pattern must have length >= 1")
        opts = _PlanOpts()
        opts.family = FAMILIES[family]
        opts.sigma_hint = 0
        opts.anchor_words = int(anchor_words)
        hist_arr = None
        if hist is not None:
            hist_arr = np.ascontiguousarray(np.asarray(hist, dtype=np.int64).reshape(256))
            opts.hist = hist_arr.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
        h = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(p, len(p))
        _check(L.mb_plan_create(ctypes.addressof(buf), len(p), ctypes.byref(opts), ctypes.byref(h)))
        self._h = h
        self.pattern = p
        self.m = len(p)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.mb_plan_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def info(self) -> PlanInfo:
        i = _PlanInfo()
        _check(load_library().mb_plan_info(self._h, ctypes.byref(i)))
        return PlanInfo(i.m, FAMILY_NAMES.get(i.family, str(i.family)), i.anchor, i.delta, i.period, bool(i.periodic),
                        i.stride, i.gram, i.words)

    # -- H1 host tables (bit-identical to the reference's functions) --
    def horspool_table(self) -> list[int]:
        out = np.empty(256, dtype=np.int64)
        _check(load_library().mb_plan_horspool(self._h, out.ctypes.data))
        return out.tolist()

    def sunday_table(self) -> list[int]:
        out = np.empty(256, dtype=np.int64)
        _check(load_library().mb_plan_sunday(self._h, out.ctypes.data))
        return out.tolist()

    def forward_masks(self) -> list[int]:
        words = (self.m + 63) // 64
        out = np.zeros(256 * words, dtype=np.uint64)
        _check(load_library().mb_plan_fwd_masks(self._h, out.ctypes.data, words))
        res = []
        for c in range(256):
            v = 0
            for w in range(words - 1, -1, -1):
                v = (v << 64) | int(out[c * words + w])
            res.append(v)
        return res

    def kmp_failure(self) -> list[int]:
        out = np.empty(self.m + 1, dtype=np.int64)
        _check(load_library().mb_plan_kmp(self._h, out.ctypes.data))
        return out.tolist()

    def gram_hashes(self, q: int) -> list[int]:
        out = np.empty(max(self.m - q + 1, 1), dtype=np.uint32)
        _check(load_library().mb_plan_gram_hash(self._h, q, out.ctypes.data))
        return out[: self.m - q + 1].tolist()


class Context:
    """Per-thread device workspace (look-back flags, tile tickets)."""

    def __init__(self, device: int = 0):
        L = load_library()
        h = ctypes.c_void_p()
        _check(L.mb_ctx_create(device, ctypes.byref(h)))
        self._h = h
        self.device = device

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.mb_ctx_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h


_tls = threading.local()


def context(device: int | None = None) -> Context:
    import torch

    if not torch.cuda.is_available():
        raise EngineError("no CUDA device: the B200 engine has no CPU fallback")
    dev = torch.cuda.current_device() if device is None else device
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    c = ctxs.get(dev)
    if c is None:
        with torch.cuda.device(dev):
            c = ctxs[dev] = Context(dev)
    return c


def _stream_handle(stream=None, device=None):
    import torch

    s = torch.cuda.current_stream(device) if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _dev_index(t) -> int:
    return t.device.index if t.device.index is not None else 0


def _wait(stream, device):
    """Before a host read of a search result: a search on a stream other than
    the device's current one is not ordered before .item()/.cpu() (which sync
    only the current stream)."""
    import torch

    if stream is not None and stream != torch.cuda.current_stream(device):
        stream.synchronize()


def to_device_text(text, device=None):
    """bytes / bytearray / memoryview / numpy / torch -> contiguous uint8 CUDA tensor
    (zero-copy when it already is one)."""
    import torch

    if isinstance(text, torch.Tensor):
        t = text
        if t.dtype != torch.uint8:
            raise TypeError("text tensor must be uint8")
        t = t.reshape(-1)
        if not t.is_cuda:
            t = t.to("cuda" if device is None else device, non_blocking=False)
        return t.contiguous()
    if isinstance(text, np.ndarray):
        arr = np.ascontiguousarray(text, dtype=np.uint8).reshape(-1)
    else:
        mv = memoryview(text)
        if mv.ndim != 1 or mv.itemsize != 1:
            mv = mv.cast("B")
        arr = np.frombuffer(mv, dtype=np.uint8)
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    out = torch.empty(arr.size, dtype=torch.uint8, device=dev)
    if arr.size:
        out.copy_(torch.from_numpy(arr.copy() if not arr.flags.writeable else arr))
    return out


def _take(out, c, stream, device):
    """Copy of out[:c] ordered after the search: on the search's stream, which
    is then drained, so the next search into the shared buffer cannot overtake it."""
    import torch

    if stream is None or stream == torch.cuda.current_stream(device):
        return out[:c].clone()
    with torch.cuda.stream(stream):
        res = out[:c].clone()
    stream.synchronize()
    return res


class _OutBuf:
    """Per-thread, per-device growable int64 output buffers."""

    def __init__(self):
        self.t = {}

    def get(self, cap, device):
        import torch

        t = self.t.get(device.index)
        if t is None or t.numel() < cap:
            t = self.t[device.index] = torch.empty(max(cap, 1 << 16), dtype=torch.int64, device=device)
        return t


def _outbuf() -> _OutBuf:
    b = getattr(_tls, "outbuf", None)
    if b is None:
        b = _tls.outbuf = _OutBuf()
    return b


def find_into(plan: Plan, d_text, out, count, stream=None):
    """Asynchronous: positions -> out (int64 CUDA tensor or None), total -> count
    (1-element int64 CUDA tensor).  Runs on the text's device (its context,
    its current stream unless `stream` is given).  Returns nothing; caller syncs."""
    import torch

    L = load_library()
    dev = _dev_index(d_text)
    with torch.cuda.device(dev):
        ctx = context(dev)
        cap = 0 if out is None else out.numel()
        _check(L.mb_find(ctx.handle, plan.handle, ctypes.c_void_p(d_text.data_ptr() if d_text.numel() else 0),
                         d_text.numel(), ctypes.c_void_p(out.data_ptr() if out is not None else 0), cap,
                         ctypes.c_void_p(count.data_ptr()), _stream_handle(stream, dev)))


def find(plan: Plan, text, stream=None):
    """All positions of plan's pattern in text as an int64 CUDA tensor (ascending)."""
    import torch

    d_text = to_device_text(text)
    dev = d_text.device
    count = torch.zeros(1, dtype=torch.int64, device=dev)
    buf = _outbuf()
    out = buf.get(1 << 16, dev)
    find_into(plan, d_text, out, count, stream)
    _wait(stream, dev)
    c = int(count.item())
    if c > out.numel():
        out = buf.get(c, dev)
        find_into(plan, d_text, out, count, stream)
        _wait(stream, dev)
        c = int(count.item())
    return _take(out, c, stream, dev)


def count(plan: Plan, text, stream=None) -> int:
    import torch

    d_text = to_device_text(text)
    cnt = torch.zeros(1, dtype=torch.int64, device=d_text.device)
    find_into(plan, d_text, None, cnt, stream)
    _wait(stream, d_text.device)
    return int(cnt.item())


class Batch:
    """Prepared batch (mb_batch_create): device params + multi-pattern tables of
    K plans built once, reused for every text -- compile once, search many."""

    def __init__(self, plans):
        L = load_library()
        self.plans = list(plans)  # keep the plans alive for the batch's lifetime
        K = len(self.plans)
        arr = (ctypes.c_void_p * K)(*[p.handle.value for p in self.plans])
        h = ctypes.c_void_p()
        _check(L.mb_batch_create(arr, K, ctypes.byref(h)))
        self._h = h

    def __len__(self):
        return len(self.plans)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.mb_batch_destroy(h)
            self._h = None


def find_batch_into(plans, d_text, out, offsets, stream=None):
    import torch

    L = load_library()
    dev = _dev_index(d_text)
    with torch.cuda.device(dev):
        ctx = context(dev)
        cap = 0 if out is None else out.numel()
        tp = ctypes.c_void_p(d_text.data_ptr() if d_text.numel() else 0)
        op = ctypes.c_void_p(out.data_ptr() if out is not None else 0)
        if isinstance(plans, Batch):
            _check(L.mb_find_batch_prepared(ctx.handle, plans._h, tp, d_text.numel(), op, cap,
                                            ctypes.c_void_p(offsets.data_ptr()), _stream_handle(stream, dev)))
            return
        K = len(plans)
        arr = (ctypes.c_void_p * K)(*[p.handle.value for p in plans])
        _check(L.mb_find_batch(ctx.handle, arr, K, tp, d_text.numel(), op, cap,
                               ctypes.c_void_p(offsets.data_ptr()), _stream_handle(stream, dev)))


def find_batch(plans, text, stream=None):
    """One text against K plans: (positions int64 CUDA tensor, offsets int64 CPU
    tensor of K+1) -- CSR, pattern k at positions[offsets[k]:offsets[k+1]]."""
    import torch

    d_text = to_device_text(text)
    dev = d_text.device
    K = len(plans)
    offsets = torch.zeros(K + 1, dtype=torch.int64, device=dev)
    buf = _outbuf()
    out = buf.get(1 << 16, dev)
    find_batch_into(plans, d_text, out, offsets, stream)
    _wait(stream, dev)
    offs = offsets.cpu()
    total = int(offs[-1])
    if total > out.numel():
        out = buf.get(total, dev)
        find_batch_into(plans, d_text, out, offsets, stream)
        _wait(stream, dev)
        offs = offsets.cpu()
    return _take(out, total, stream, dev), offs


def histogram(text, stream=None):
    """K0: 256-bin byte histogram of the text on the device (int64 CUDA tensor)."""
    import torch

    d_text = to_device_text(text)
    dev = _dev_index(d_text)
    with torch.cuda.device(dev):
        hist = torch.zeros(256, dtype=torch.int64, device=d_text.device)
        _check(load_library().mb_histogram(context(dev).handle,
                                           ctypes.c_void_p(d_text.data_ptr() if d_text.numel() else 0),
                                           d_text.numel(), ctypes.c_void_p(hist.data_ptr()),
                                           _stream_handle(stream, dev)))
    _wait(stream, d_text.device)
    return hist


def search_host(pattern: bytes, text_np: np.ndarray, cap: int | None = None) -> np.ndarray:
    """The C-ABI host-buffer entry (mb_search_host): host text in, host positions out."""
    L = load_library()
    ctx = context()
    p = bytes(pattern)
    t = np.ascontiguousarray(text_np, dtype=np.uint8).reshape(-1)
    cap = 1 << 16 if cap is None else cap
    while True:
        out = np.empty(max(cap, 1), dtype=np.int64)
        cnt = ctypes.c_int64(0)
        pb = ctypes.create_string_buffer(p, len(p))
        rc = L.mb_search_host(ctx.handle, ctypes.addressof(pb), len(p),
                              ctypes.c_void_p(t.ctypes.data if t.size else 0), t.size,
                              ctypes.c_void_p(out.ctypes.data), cap, ctypes.byref(cnt))
        if rc == MB_EOVERFLOW:
            cap = cnt.value
            continue
        _check(rc)
        return out[: cnt.value]


def search_batch_host(patterns, text_np: np.ndarray, h_out: np.ndarray, h_offsets: np.ndarray) -> int:
    """mb_search_batch_host into caller-provided host buffers; returns rc (EOVERFLOW allowed)."""
    L = load_library()
    ctx = context()
    K = len(patterns)
    bufs = [ctypes.create_string_buffer(bytes(p), len(p)) for p in patterns]
    parr = (ctypes.c_void_p * K)(*[ctypes.addressof(b) for b in bufs])
    ms = (ctypes.c_int64 * K)(*[len(p) for p in patterns])
    t = text_np
    rc = L.mb_search_batch_host(ctx.handle, parr, ms, K, ctypes.c_void_p(t.ctypes.data if t.size else 0), t.size,
                                ctypes.c_void_p(h_out.ctypes.data), h_out.size, ctypes.c_void_p(h_offsets.ctypes.data))
    if rc not in (MB_OK, MB_EOVERFLOW):
        _check(rc)
    return rc
