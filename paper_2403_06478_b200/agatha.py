"""Thin ctypes binding of libagatha.so (include/agatha.h).  Argument marshalling only.

Every step of the path (packing, planning, the wavefront alignment, the result write)
runs in the library's sm_100a kernels.  This module only turns numpy arrays / torch
tensors into pointers and back.  It raises if the library is missing: there is no
CPU fallback.

Names follow the C ABI: ``agatha_align_batch`` -> ``align_batch`` etc.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libagatha.so")

OK, EINVAL, EEMPTY, ECHAR, ERANGE, ECUDA, ENOMEM = 0, -1, -2, -3, -4, -5, -6
MEM_HOST, MEM_DEVICE, OUT_DEVICE = 0, 1, 2
N_REJECT, N_MAP, PACK_REVERSE, ORDER_INPUT, FORCE_32BIT, SINGLE_TIER = 0, 4, 8, 16, 32, 64
STATIC_ASSIGN = 128  # ablation: no work queue, warp u takes order positions u, u + W, ...

RESULT_DTYPE = np.dtype([("score", "<i4"), ("ref_end", "<i4"), ("query_end", "<i4"),
                         ("zdrop_antidiag", "<i4"), ("cells", "<i8")])


class AgathaError(RuntimeError):
    def __init__(self, code: int, what: str = ""):
        self.code = code
        super().__init__(f"{what}: {strerror(code)} ({code})" if what else f"{strerror(code)} ({code})")


class Params(ctypes.Structure):
    """agatha_params_t.  Penalties are positive numbers; negative band / zdrop disable."""
    _fields_ = [("match", ctypes.c_int32), ("mismatch", ctypes.c_int32),
                ("ambig", ctypes.c_int32), ("gap_open", ctypes.c_int32),
                ("gap_extend", ctypes.c_int32), ("band_left", ctypes.c_int32),
                ("band_right", ctypes.c_int32), ("zdrop", ctypes.c_int32),
                ("variant", ctypes.c_int32)]


VAR_GATE_GE, VAR_ORIGIN_MAX, VAR_CHECK_LAST = 1, 2, 4


class Batch(ctypes.Structure):
    _fields_ = [("ref", ctypes.c_void_p), ("qry", ctypes.c_void_p), ("ref_off", ctypes.c_void_p),
                ("qry_off", ctypes.c_void_p), ("n_pairs", ctypes.c_uint64),
                ("flags", ctypes.c_uint32), ("queue", ctypes.c_void_p), ("ends", ctypes.c_void_p)]


class Stats(ctypes.Structure):
    _fields_ = [("h2d_ms", ctypes.c_float), ("prep_ms", ctypes.c_float),
                ("align_ms", ctypes.c_float), ("d2h_ms", ctypes.c_float),
                ("slots_per_lane", ctypes.c_int32), ("grid_blocks", ctypes.c_int32),
                ("kernel_launches", ctypes.c_int32), ("library_launches", ctypes.c_int32),
                ("packed16", ctypes.c_int32), ("warps_per_pair", ctypes.c_int32),
                ("tier_pairs", ctypes.c_int32 * 3), ("input_chunks", ctypes.c_int32),
                ("lpt_from_chunk", ctypes.c_int32), ("pin_off", ctypes.c_int32),
                ("rebase_iters", ctypes.c_int32), ("pin_off8", ctypes.c_int32)]

    def as_dict(self):
        return {k: (list(v) if k == "tier_pairs" else v)
                for k, v in ((k, getattr(self, k)) for k, _ in self._fields_)}


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libagatha.so not built ({LIB_PATH}); run __graft_entry__.build()")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i32, u64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint64
    lib.agatha_ctx_create.argtypes = [ctypes.POINTER(vp), ctypes.c_int]
    lib.agatha_ctx_destroy.argtypes = [vp]
    lib.agatha_ctx_destroy.restype = None
    lib.agatha_align_batch.argtypes = [vp, ctypes.POINTER(Batch), ctypes.POINTER(Params), vp, vp]
    lib.agatha_pack4.argtypes = [vp, vp, u64, vp, ctypes.c_uint32, vp]
    lib.agatha_plan.argtypes = [vp, ctypes.POINTER(Batch), ctypes.POINTER(Params), vp, vp, vp]
    lib.agatha_localmax_trace.argtypes = [vp, ctypes.POINTER(Batch), ctypes.POINTER(Params), u64,
                                          vp, vp, ctypes.c_int64, vp]
    lib.agatha_get_stats.argtypes = [vp, ctypes.POINTER(Stats)]
    lib.agatha_strerror.argtypes = [ctypes.c_int]
    lib.agatha_strerror.restype = ctypes.c_char_p
    lib.agatha_version.restype = ctypes.c_int
    lib.agatha_queue_create.argtypes = [vp, ctypes.POINTER(vp), ctypes.c_char_p]
    lib.agatha_queue_open.argtypes = [vp, ctypes.c_char_p, ctypes.POINTER(vp)]
    lib.agatha_queue_reset.argtypes = [vp, vp, vp]
    lib.agatha_queue_close.argtypes = [vp, vp, ctypes.c_int]
    lib.agatha_align_federated.argtypes = [vp, ctypes.POINTER(Batch), ctypes.c_int, ctypes.POINTER(Params),
                                           vp, vp, ctypes.c_uint32, vp]
    lib.agatha_ipc_alloc.argtypes = [vp, u64, ctypes.POINTER(vp), ctypes.c_char_p]
    lib.agatha_ipc_open.argtypes = [vp, ctypes.c_char_p, ctypes.POINTER(vp)]
    lib.agatha_ipc_close.argtypes = [vp, vp, ctypes.c_int]
    return lib


_lib = _load()

# Every symbol include/agatha.h declares (checked by tests/test_abi.py).
EXPORTS = ("agatha_ctx_create", "agatha_ctx_destroy", "agatha_align_batch", "agatha_pack4",
           "agatha_plan", "agatha_localmax_trace", "agatha_get_stats", "agatha_strerror",
           "agatha_version", "agatha_queue_create", "agatha_queue_open", "agatha_queue_reset",
           "agatha_queue_close", "agatha_align_federated", "agatha_ipc_alloc", "agatha_ipc_open",
           "agatha_ipc_close")


def lib() -> ctypes.CDLL:
    return _lib


def strerror(code: int) -> str:
    return _lib.agatha_strerror(code).decode()


def version() -> int:
    return int(_lib.agatha_version())


def make_params(match=2, mismatch=4, ambig=None, gap_open=4, gap_extend=2, band_left=-1,
                band_right=-1, zdrop=-1, variant=0, **_ignored) -> Params:
    return Params(match, mismatch, mismatch if ambig is None else ambig, gap_open, gap_extend,
                  band_left, band_right, zdrop, variant)


def params_from(obj) -> Params:
    if isinstance(obj, Params):
        return obj
    if isinstance(obj, dict):
        return make_params(**obj)
    d = {k: getattr(obj, k) for k in (
        "match", "mismatch", "ambig", "gap_open", "gap_extend", "band_left", "band_right", "zdrop")}
    d["variant"] = getattr(obj, "variant", 0)
    return make_params(**d)


def _stream_ptr(stream) -> Optional[int]:
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except Exception:  # pragma: no cover
            pass
        return None
    return int(getattr(stream, "cuda_stream", stream))


class Context:
    """agatha_ctx_t on one CUDA device (owns the library's device scratch)."""

    def __init__(self, device: int = 0):
        h = ctypes.c_void_p()
        rc = _lib.agatha_ctx_create(ctypes.byref(h), int(device))
        if rc != OK:
            raise AgathaError(rc, "agatha_ctx_create")
        self.handle = h
        self.device = device

    def close(self):
        if getattr(self, "handle", None):
            _lib.agatha_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def stats(self) -> dict:
        s = Stats()
        _lib.agatha_get_stats(self.handle, ctypes.byref(s))
        return s.as_dict()


class SharedQueue:
    """A pair counter shared by several contexts, processes or GPUs (agatha_queue_*;
    cross-GPU dynamic balancing, NEXT #1).  ``SharedQueue.create(ctx)`` allocates it and
    exposes ``handle`` (64 bytes, to send to the other participants);
    ``SharedQueue.open(ctx, handle)`` maps one created by another process.  Pass
    ``queue=`` to align_batch."""

    def __init__(self, ctx: Context, ptr: int, handle: bytes, opened: bool):
        self.ctx, self.ptr, self.handle, self.opened = ctx, ptr, handle, opened

    @classmethod
    def create(cls, ctx: Context) -> "SharedQueue":
        q = ctypes.c_void_p()
        h = ctypes.create_string_buffer(64)
        rc = _lib.agatha_queue_create(ctx.handle, ctypes.byref(q), h)
        if rc != OK:
            raise AgathaError(rc, "agatha_queue_create")
        return cls(ctx, int(q.value), h.raw, False)

    @classmethod
    def open(cls, ctx: Context, handle: bytes) -> "SharedQueue":
        q = ctypes.c_void_p()
        rc = _lib.agatha_queue_open(ctx.handle, bytes(handle), ctypes.byref(q))
        if rc != OK:
            raise AgathaError(rc, "agatha_queue_open")
        return cls(ctx, int(q.value), bytes(handle), True)

    def reset(self, stream=None):
        rc = _lib.agatha_queue_reset(self.ctx.handle, self.ptr, _stream_ptr(stream))
        if rc != OK:
            raise AgathaError(rc, "agatha_queue_reset")

    def close(self):
        if self.ptr:
            _lib.agatha_queue_close(self.ctx.handle, self.ptr, int(self.opened))
            self.ptr = 0


class IpcBuffer:
    """Device memory another process can map (agatha_ipc_*): ``IpcBuffer.alloc(ctx, n)``
    allocates n bytes and exposes ``handle`` (64 bytes); ``IpcBuffer.open(ctx, handle, n)``
    maps another process's buffer.  ``ptr`` is the device address in this process."""

    def __init__(self, ctx: Context, ptr: int, nbytes: int, handle: bytes, opened: bool):
        self.ctx, self.ptr, self.nbytes, self.handle, self.opened = ctx, ptr, nbytes, handle, opened

    @classmethod
    def alloc(cls, ctx: Context, nbytes: int) -> "IpcBuffer":
        q = ctypes.c_void_p()
        h = ctypes.create_string_buffer(64)
        rc = _lib.agatha_ipc_alloc(ctx.handle, max(int(nbytes), 1), ctypes.byref(q), h)
        if rc != OK:
            raise AgathaError(rc, "agatha_ipc_alloc")
        return cls(ctx, int(q.value), int(nbytes), h.raw, False)

    @classmethod
    def open(cls, ctx: Context, handle: bytes, nbytes: int) -> "IpcBuffer":
        q = ctypes.c_void_p()
        rc = _lib.agatha_ipc_open(ctx.handle, bytes(handle), ctypes.byref(q))
        if rc != OK:
            raise AgathaError(rc, "agatha_ipc_open")
        return cls(ctx, int(q.value), int(nbytes), bytes(handle), True)

    def copy_from_host(self, arr, offset: int = 0, stream=None):
        """Host -> this buffer (cudaMemcpyAsync on ``stream``, plumbing only)."""
        from cuda.bindings import runtime as rt

        a = np.ascontiguousarray(arr)
        if a.nbytes + offset > self.nbytes:
            raise ValueError("copy exceeds the buffer")
        st = _stream_ptr(stream) or 0
        err, = rt.cudaMemcpyAsync(self.ptr + offset, a.ctypes.data, a.nbytes,
                                  rt.cudaMemcpyKind.cudaMemcpyHostToDevice, st)
        if err != rt.cudaError_t.cudaSuccess:
            raise AgathaError(ECUDA, f"cudaMemcpyAsync: {err}")
        if stream is None:
            rt.cudaStreamSynchronize(0)

    def close(self):
        if self.ptr:
            _lib.agatha_ipc_close(self.ctx.handle, self.ptr, int(self.opened))
            self.ptr = 0


class DevicePtr:
    """A raw device address (e.g. inside an IpcBuffer) usable where align_batch /
    align_federated take a device array."""

    is_cuda = True

    def __init__(self, ptr: int, n: int):
        self.ptr, self.n = int(ptr), int(n)

    def data_ptr(self) -> int:
        return self.ptr

    def __len__(self) -> int:
        return self.n


def align_federated(ctx: Context, owners, params, out, queue: Optional["SharedQueue"] = None,
                    flags: int = 0, stream=None):
    """agatha_align_federated.  ``owners``: list of (ref, ref_off, qry, qry_off) device
    arrays (torch CUDA tensors or DevicePtr), one per owner, in global order; ``out``: a
    CUDA uint8 tensor of 24 * total pairs."""
    arr = (Batch * len(owners))()
    for o, (ref, ref_off, qry, qry_off) in enumerate(owners):
        arr[o] = make_batch(ref, ref_off, qry, qry_off)
    p = params_from(params)
    rc = _lib.agatha_align_federated(ctx.handle, arr, len(owners), ctypes.byref(p), _ptr(out),
                                     queue.ptr if queue is not None else None, flags, _stream_ptr(stream))
    if rc != OK:
        raise AgathaError(rc, "agatha_align_federated")
    return out


def _ptr(a) -> int:
    if a is None:
        return 0
    if hasattr(a, "data_ptr"):
        return int(a.data_ptr())
    return int(a.ctypes.data)


def _is_cuda(a) -> bool:
    return hasattr(a, "is_cuda") and bool(a.is_cuda)


def make_batch(ref, ref_off, qry, qry_off, flags: int = 0) -> Batch:
    """Batch from numpy arrays (host) or torch CUDA tensors (device)."""
    n_pairs = int(len(ref_off)) - 1
    dev = _is_cuda(ref)
    if dev != _is_cuda(qry) or dev != _is_cuda(ref_off) or dev != _is_cuda(qry_off):
        raise ValueError("all batch arrays must be on the same side (host or device)")
    if dev:
        flags |= MEM_DEVICE
    return Batch(_ptr(ref), _ptr(qry), _ptr(ref_off), _ptr(qry_off), n_pairs, flags)


# NEXT #4 end scores (agatha_ends_t): mqe / mqe_i, mte / mte_j, end_score; absent -> NO_SCORE, -1
ENDS_DTYPE = np.dtype([("mqe", "<i4"), ("mqe_i", "<i4"), ("mte", "<i4"), ("mte_j", "<i4"),
                       ("end_score", "<i4"), ("reserved", "<i4")])
NO_SCORE = -(1 << 30)


def align_batch(ctx: Context, ref, ref_off, qry, qry_off, params, out=None, flags: int = 0,
                stream=None, queue: Optional["SharedQueue"] = None, ends=None):
    """agatha_align_batch.  Returns ``out`` (a numpy RESULT_DTYPE array for host outputs,
    or the given CUDA uint8/int tensor of 24*n_pairs bytes for device outputs).  With a
    ``queue`` (SharedQueue) only the pairs this call claims are aligned; the other rows of
    ``out`` are zero."""
    b = make_batch(ref, ref_off, qry, qry_off, flags)
    if queue is not None:
        b.queue = queue.ptr
    if ends is not None:  # same side as `out`: numpy ENDS_DTYPE array, or CUDA bytes
        b.ends = _ptr(ends)
    p = params_from(params)
    if out is None:
        out = np.zeros(b.n_pairs, RESULT_DTYPE)
    if _is_cuda(out):
        b.flags |= OUT_DEVICE
    rc = _lib.agatha_align_batch(ctx.handle, ctypes.byref(b), ctypes.byref(p), _ptr(out),
                                 _stream_ptr(stream))
    if rc != OK:
        raise AgathaError(rc, "agatha_align_batch")
    return out


def align_pairs(ctx: Context, pairs, params, flags: int = 0, stream=None):
    """Convenience: align a ``synth.Pairs``-like object (host arrays)."""
    return align_batch(ctx, pairs.ref, pairs.ref_off, pairs.qry, pairs.qry_off, params,
                       flags=flags, stream=stream)


def align_pairs_ends(ctx: Context, pairs, params, flags: int = 0, stream=None):
    """align_pairs plus the NEXT #4 end scores: ``(results, ends)`` (host arrays)."""
    ends = np.zeros(pairs.n_pairs, ENDS_DTYPE)
    res = align_batch(ctx, pairs.ref, pairs.ref_off, pairs.qry, pairs.qry_off, params,
                      flags=flags, stream=stream, ends=ends)
    return res, ends


def align_pairs_q(ctx: Context, pairs, params, out, queue: "SharedQueue", stream=None, flags: int = 0):
    """align_pairs into ``out`` claiming pairs from a SharedQueue (NEXT #1)."""
    return align_batch(ctx, pairs.ref, pairs.ref_off, pairs.qry, pairs.qry_off, params, out=out,
                       flags=flags, stream=stream, queue=queue)


def device_results(out_tensor):
    """View a device result buffer (torch uint8, 24*n bytes) as a numpy RESULT_DTYPE array."""
    return out_tensor.cpu().numpy().view(RESULT_DTYPE)


def pack4(ctx: Context, ascii_dev, words_dev, flags: int = 0, stream=None) -> int:
    """agatha_pack4 on device buffers; returns the rc (raises on CUDA errors only)."""
    rc = _lib.agatha_pack4(ctx.handle, _ptr(ascii_dev), int(ascii_dev.numel()), _ptr(words_dev),
                           flags, _stream_ptr(stream))
    if rc in (ECUDA, ENOMEM, EINVAL):
        raise AgathaError(rc, "agatha_pack4")
    return rc


def plan(ctx: Context, ref, ref_off, qry, qry_off, params, order_dev, nominal_dev, stream=None):
    """agatha_plan (device inputs and outputs)."""
    b = make_batch(ref, ref_off, qry, qry_off)
    p = params_from(params)
    rc = _lib.agatha_plan(ctx.handle, ctypes.byref(b), ctypes.byref(p), _ptr(order_dev),
                          _ptr(nominal_dev), _stream_ptr(stream))
    if rc != OK:
        raise AgathaError(rc, "agatha_plan")


def localmax_trace(ctx: Context, ref, ref_off, qry, qry_off, params, pair: int, cap: int,
                   flags: int = 0, stream=None):
    """agatha_localmax_trace: (score[c], i[c]) of Eq. 5 for one pair, c in [0, cap)."""
    b = make_batch(ref, ref_off, qry, qry_off, flags)
    p = params_from(params)
    score = np.zeros(cap, np.int32)
    ri = np.zeros(cap, np.int32)
    rc = _lib.agatha_localmax_trace(ctx.handle, ctypes.byref(b), ctypes.byref(p), pair,
                                    _ptr(score), _ptr(ri), cap, _stream_ptr(stream))
    if rc != OK:
        raise AgathaError(rc, "agatha_localmax_trace")
    return score, ri
