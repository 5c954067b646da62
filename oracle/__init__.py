"""CPU oracle for guided (banded + Z-drop) affine-gap extension alignment.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this package.
The CUDA product path (``paper_2403_06478_b200``) never imports it, and the two
share no code: this package compiles its own plain C file (``agatha_oracle.c``)
with gcc and declares its own ctypes types.

Functions
---------
``align_batch``   all pairs of a batch (multi-threaded, longest first)
``align_one``     one pair, optionally with the per-anti-diagonal local-max trace
``pack4``         the plain definition of 4-bit packing (§2.2, l.279-285)
``nominal_cells`` in-band in-table cell count of an un-terminated pair

Each C function cites the PAPER.md passage it transcribes.  ``bruteforce`` (pure
Python path enumeration) is the independent pin used to write ``tests/golden``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "agatha_oracle.c")
_LIB = os.path.join(_HERE, "libagatha_oracle.so")

OK, EINVAL, EEMPTY, ECHAR, ENOMEM = 0, -1, -2, -3, -6

RESULT_DTYPE = np.dtype([("score", "<i4"), ("ref_end", "<i4"), ("query_end", "<i4"),
                         ("zdrop_antidiag", "<i4"), ("cells", "<i8")])


class Params(ctypes.Structure):
    _fields_ = [("match", ctypes.c_int32), ("mismatch", ctypes.c_int32),
                ("ambig", ctypes.c_int32), ("gap_open", ctypes.c_int32),
                ("gap_extend", ctypes.c_int32), ("band_left", ctypes.c_int32),
                ("band_right", ctypes.c_int32), ("zdrop", ctypes.c_int32),
                ("variant", ctypes.c_int32)]


VAR_GATE_GE, VAR_ORIGIN_MAX, VAR_CHECK_LAST = 1, 2, 4


class _Result(ctypes.Structure):
    _fields_ = [("score", ctypes.c_int32), ("ref_end", ctypes.c_int32),
                ("query_end", ctypes.c_int32), ("zdrop_antidiag", ctypes.c_int32),
                ("cells", ctypes.c_int64)]


class _Trace(ctypes.Structure):
    _fields_ = [("score", ctypes.POINTER(ctypes.c_int32)), ("i", ctypes.POINTER(ctypes.c_int32)),
                ("cap", ctypes.c_int64)]


def make_params(match=2, mismatch=4, ambig=None, gap_open=4, gap_extend=2, band_left=-1,
                band_right=-1, zdrop=-1, variant=0, **_ignored) -> Params:
    return Params(match, mismatch, mismatch if ambig is None else ambig, gap_open, gap_extend,
                  band_left, band_right, zdrop, variant)


def params_from(obj) -> Params:
    """Accept an oracle.Params, a dict or any object with the eight scoring attributes."""
    if isinstance(obj, Params):
        return obj
    if isinstance(obj, dict):
        return make_params(**obj)
    d = {k: getattr(obj, k) for k in (
        "match", "mismatch", "ambig", "gap_open", "gap_extend", "band_left", "band_right", "zdrop")}
    d["variant"] = getattr(obj, "variant", 0)
    return make_params(**d)


_lib: Optional[ctypes.CDLL] = None


def build(force: bool = False) -> str:
    """Compile the oracle (plain C, gcc -O2).  Building the checker is not using it."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = f"{_LIB}.{os.getpid()}.tmp"  # replaced atomically: a running user keeps the old one
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", tmp, _SRC,
                               "-lpthread"])
        os.replace(tmp, _LIB)
    return _LIB


def _load() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        lib.oracle_align_one.argtypes = [ctypes.c_char_p, ctypes.c_int64, ctypes.c_char_p,
                                         ctypes.c_int64, ctypes.POINTER(Params),
                                         ctypes.POINTER(_Result), ctypes.POINTER(_Trace)]
        lib.oracle_align_batch.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_uint64,
                                           ctypes.POINTER(Params), ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_int]
        lib.oracle_align_one_ends.argtypes = [ctypes.c_char_p, ctypes.c_int64, ctypes.c_char_p,
                                              ctypes.c_int64, ctypes.POINTER(Params),
                                              ctypes.POINTER(_Result), ctypes.c_void_p, ctypes.c_void_p]
        lib.oracle_align_batch_ends.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                                ctypes.c_void_p, ctypes.c_uint64, ctypes.POINTER(Params),
                                                ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        lib.oracle_nominal_cells.argtypes = [ctypes.c_int64] * 4
        lib.oracle_nominal_cells.restype = ctypes.c_int64
        lib.oracle_pack4.argtypes = [ctypes.c_char_p, ctypes.c_int64, ctypes.c_void_p,
                                     ctypes.c_int, ctypes.c_int]
        lib.oracle_validate.argtypes = [ctypes.POINTER(Params)]
        _lib = lib
    return _lib


def _b(s) -> bytes:
    return s.encode() if isinstance(s, str) else bytes(s)


def align_one(R, Q, params, trace: bool = False):
    """Return ``(rc, result_tuple[, (local_scores, local_i)])`` for one pair."""
    R, Q = _b(R), _b(Q)
    p = params_from(params)
    res = _Result()
    tr = None
    if trace:
        cap = len(R) + len(Q) + 1
        ts = np.zeros(cap, np.int32)
        ti = np.full(cap, -1, np.int32)
        tr = _Trace(ts.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                    ti.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), cap)
    rc = _load().oracle_align_one(R, len(R), Q, len(Q), ctypes.byref(p), ctypes.byref(res),
                                  ctypes.byref(tr) if tr is not None else None)
    out = (res.score, res.ref_end, res.query_end, res.zdrop_antidiag, res.cells)
    if trace:
        return rc, out, (ts, ti)
    return rc, out


def align_batch(pairs, params, threads: Optional[int] = None):
    """Align every pair of ``pairs`` (a ``synth.Pairs``).  Returns (rc, results, status)."""
    p = params_from(params)
    n = pairs.n_pairs
    out = np.zeros(n, RESULT_DTYPE)
    status = np.zeros(n, np.int32)
    if n == 0:
        return EEMPTY, out, status
    ref_off = np.ascontiguousarray(pairs.ref_off, np.uint64)
    qry_off = np.ascontiguousarray(pairs.qry_off, np.uint64)
    ref = np.ascontiguousarray(pairs.ref, np.uint8)
    qry = np.ascontiguousarray(pairs.qry, np.uint8)
    rc = _load().oracle_align_batch(ref.ctypes.data, ref_off.ctypes.data, qry.ctypes.data,
                                    qry_off.ctypes.data, n, ctypes.byref(p), out.ctypes.data,
                                    status.ctypes.data, threads or (os.cpu_count() or 1))
    return rc, out, status


# NEXT #4 end scores (reading R19): mqe / mqe_i (query end), mte / mte_j (reference end),
# end_score = H(m, n); absent -> NO_SCORE and position -1.
ENDS_DTYPE = np.dtype([("mqe", "<i4"), ("mqe_i", "<i4"), ("mte", "<i4"), ("mte_j", "<i4"),
                       ("end_score", "<i4"), ("reserved", "<i4")])
NO_SCORE = -(1 << 30)


def align_one_ends(R, Q, params):
    """``(rc, result_tuple, ends_tuple)`` for one pair (ends = mqe, mqe_i, mte, mte_j, end_score)."""
    R, Q = _b(R), _b(Q)
    p = params_from(params)
    res = _Result()
    ends = np.zeros(1, ENDS_DTYPE)
    rc = _load().oracle_align_one_ends(R, len(R), Q, len(Q), ctypes.byref(p), ctypes.byref(res), None,
                                       ends.ctypes.data)
    out = (res.score, res.ref_end, res.query_end, res.zdrop_antidiag, res.cells)
    return rc, out, tuple(ends[0].tolist())[:5]


def align_batch_ends(pairs, params, threads: Optional[int] = None):
    """align_batch plus each pair's end scores: ``(rc, results, ends, status)``."""
    p = params_from(params)
    n = pairs.n_pairs
    out = np.zeros(n, RESULT_DTYPE)
    ends = np.zeros(n, ENDS_DTYPE)
    status = np.zeros(n, np.int32)
    if n == 0:
        return EEMPTY, out, ends, status
    ref_off = np.ascontiguousarray(pairs.ref_off, np.uint64)
    qry_off = np.ascontiguousarray(pairs.qry_off, np.uint64)
    ref = np.ascontiguousarray(pairs.ref, np.uint8)
    qry = np.ascontiguousarray(pairs.qry, np.uint8)
    rc = _load().oracle_align_batch_ends(ref.ctypes.data, ref_off.ctypes.data, qry.ctypes.data,
                                         qry_off.ctypes.data, n, ctypes.byref(p), out.ctypes.data,
                                         ends.ctypes.data, status.ctypes.data, threads or (os.cpu_count() or 1))
    return rc, out, ends, status


def nominal_cells(m: int, n: int, band_left: int, band_right: int) -> int:
    return int(_load().oracle_nominal_cells(m, n, band_left, band_right))


def pack4(seq, reverse: bool = False, n_map: bool = False):
    """Return ``(rc, words)``: the plain 4-bit packing of ``seq`` (uint32 words)."""
    seq = _b(seq)
    words = np.zeros(max(1, (len(seq) + 7) // 8), np.uint32)
    rc = _load().oracle_pack4(seq, len(seq), words.ctypes.data, int(reverse), int(n_map))
    return rc, words


def validate(params) -> int:
    return int(_load().oracle_validate(ctypes.byref(params_from(params))))
