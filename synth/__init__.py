"""Seeded synthetic input generator shared by the oracle, the CUDA path, tests and bench.

This module holds NO alignment arithmetic: it only draws (reference window R, read Q)
pairs, as upper-case ASCII, from a counter-based RNG (``agatha_synth.c``).  The recipe
and the configurations C0..C5 follow SURVEY.md §8(d) "Synthetic inputs" and are
restated in DESIGN.md ("Input recipe").

Scoring for every configuration is the paper's example values (§2.1, lines
224-226: match +2, mismatch -4, gap open alpha=4, gap extend beta=2), with the N
penalty equal to the mismatch penalty (SPEC.md align-core design decisions).
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "agatha_synth.c")
_LIB = os.path.join(_HERE, "libagatha_synth.so")


class _Cfg(ctypes.Structure):
    _fields_ = [
        ("len_dist", ctypes.c_uint32),
        ("ref_extra_abs", ctypes.c_uint32),
        ("lo", ctypes.c_double),
        ("hi", ctypes.c_double),
        ("lo2", ctypes.c_double),
        ("hi2", ctypes.c_double),
        ("p_long", ctypes.c_double),
        ("err_lo", ctypes.c_double),
        ("err_hi", ctypes.c_double),
        ("f_sub", ctypes.c_double),
        ("f_ins", ctypes.c_double),
        ("f_del", ctypes.c_double),
        ("p_chim", ctypes.c_double),
        ("n_rate", ctypes.c_double),
        ("ref_extra_frac", ctypes.c_double),
    ]


@dataclasses.dataclass(frozen=True)
class Scoring:
    match: int = 2
    mismatch: int = 4
    ambig: int = 4
    gap_open: int = 4
    gap_extend: int = 2
    band_left: int = 100
    band_right: int = 100
    zdrop: int = 100


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    n_pairs: int
    seed: int
    len_dist: int  # 0 uniform, 1 log-uniform, 2 mixture of log-uniforms, 3 two-point mixture
    lo: float
    hi: float
    err_lo: float
    err_hi: float
    f_sub: float
    f_ins: float
    f_del: float
    p_chim: float
    scoring: Scoring
    lo2: float = 0.0
    hi2: float = 0.0
    p_long: float = 0.0
    n_rate: float = 1e-4
    ref_extra_frac: float = 0.01
    ref_extra_abs: int = 50
    description: str = ""

    def with_pairs(self, n_pairs: int) -> "Config":
        return dataclasses.replace(self, n_pairs=n_pairs)

    def _c(self) -> _Cfg:
        return _Cfg(self.len_dist, self.ref_extra_abs, self.lo, self.hi, self.lo2, self.hi2,
                    self.p_long, self.err_lo, self.err_hi, self.f_sub, self.f_ins, self.f_del,
                    self.p_chim, self.n_rate, self.ref_extra_frac)


_T = 1.0 / 3.0
CONFIGS = {
    # BASELINE.json configs[0]: the oracle finishes it in seconds.
    "C1": Config("C1", 1_000, 1, 0, 900, 1100, 0.10, 0.10, _T, _T, _T, 0.1,
                 Scoring(band_left=100, band_right=100, zdrop=100),
                 description="1,000 pairs ~1 kbp, 10% error, w=100, Z=100"),
    # configs[1]: the headline single-GPU workload (bench.py N=1).
    "C2": Config("C2", 100_000, 2, 0, 10_000, 20_000, 0.01, 0.01, 0.4, 0.3, 0.3, 0.0,
                 Scoring(band_left=500, band_right=500, zdrop=400),
                 description="100k HiFi-like pairs 10-20 kbp, 1% error, w=500, Z=400"),
    # configs[2]: ONT-like, frequent Z-drop termination.
    "C3": Config("C3", 20_000, 3, 1, 10_000, 100_000, 0.10, 0.15, 0.4, 0.25, 0.35, 0.5,
                 Scoring(band_left=500, band_right=500, zdrop=400),
                 description="20k ONT-like pairs log-U[10k,100k], 10-15% error, 50% chimeric"),
    # configs[3]: skewed lengths (10% long tail carrying ~2/3 of the cells).
    "C4": Config("C4", 1_000_000, 4, 2, 1_000, 8_000, 0.05, 0.05, _T, _T, _T, 0.1,
                 Scoring(band_left=500, band_right=500, zdrop=400),
                 lo2=30_000, hi2=100_000, p_long=0.1,
                 description="1M pairs, 90% log-U[1k,8k] + 10% log-U[30k,100k]"),
    # configs[4]: scaling sweep.
    "C5": Config("C5", 128_000, 5, 0, 10_000, 50_000, 0.05, 0.05, _T, _T, _T, 0.1,
                 Scoring(band_left=500, band_right=500, zdrop=400),
                 description="128k pairs 10-50 kbp, 5% error"),
    # Parity corpus shaped like SPEC.md's acceptance corpus: short, random.
    "C0": Config("C0", 10_000, 0, 0, 1, 512, 0.0, 0.30, _T, _T, _T, 0.3,
                 Scoring(band_left=32, band_right=32, zdrop=30),
                 description="10k parity pairs, lengths 1-512, random error"),
}


# NEXT #2: the paper's long/short study (§5.6 l.778-795):
# 4096 bp long vs 128 bp short reads mixed at a varying long percentage.  The paper
# gives no band, error or batch size; these use the C4 recipe (5% error, 10% chimeric,
# w = 500, Z = 400) with 100k pairs.
for _pct in (1, 5, 10, 25, 50):
    CONFIGS[f"LS{_pct:02d}"] = Config(
        f"LS{_pct:02d}", 100_000, 100 + _pct, 3, 128, 128, 0.05, 0.05, _T, _T, _T, 0.1,
        Scoring(band_left=500, band_right=500, zdrop=400), lo2=4096, hi2=4096, p_long=_pct / 100,
        description=f"100k pairs, {_pct}% 4096 bp + {100 - _pct}% 128 bp (PAPER.md l.786-788)")

# NEXT #3: wide bands, the C2 recipe with w = 1000 (two warps per pair)
# and w = 2000 (four warps per pair).
CONFIGS["CW1"] = dataclasses.replace(CONFIGS["C2"], name="CW1", n_pairs=20_000, seed=201,
                                     scoring=Scoring(band_left=1000, band_right=1000, zdrop=400),
                                     description="20k HiFi-like pairs 10-20 kbp, 1% error, w=1000, Z=400")
CONFIGS["CW2"] = dataclasses.replace(CONFIGS["C2"], name="CW2", n_pairs=10_000, seed=202,
                                     scoring=Scoring(band_left=2000, band_right=2000, zdrop=400),
                                     description="10k HiFi-like pairs 10-20 kbp, 1% error, w=2000, Z=400")

_lib: Optional[ctypes.CDLL] = None


# Version of the generated bytes: bump it whenever any pair of any config would change
# (tools/oracle_cache.py keys cached oracle results on it).  Additive API changes that
# leave every pair's bytes identical keep it.
GENERATOR_VERSION = "splitmix64-walk-v1"


def build(force: bool = False) -> str:
    """Compile libagatha_synth.so in-tree with gcc (plain C, no CUDA).  The library is
    replaced atomically, so a process that has the old one loaded keeps running."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = f"{_LIB}.{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", tmp, _SRC,
                               "-lm", "-lpthread"])
        os.replace(tmp, _LIB)
    return _LIB


def _load() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        u64p = ctypes.POINTER(ctypes.c_uint64)
        lib.synth_lengths.argtypes = [ctypes.POINTER(_Cfg), ctypes.c_uint64, ctypes.c_uint64,
                                      ctypes.c_uint64, u64p, u64p]
        lib.synth_fill.argtypes = [ctypes.POINTER(_Cfg), ctypes.c_uint64, ctypes.c_uint64,
                                   ctypes.c_uint64, u64p, u64p, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_int]
        lib.synth_lengths_idx.argtypes = [ctypes.POINTER(_Cfg), ctypes.c_uint64, u64p,
                                          ctypes.c_uint64, u64p, u64p]
        lib.synth_fill_idx.argtypes = [ctypes.POINTER(_Cfg), ctypes.c_uint64, u64p, ctypes.c_uint64,
                                       u64p, u64p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        _lib = lib
    return _lib


def _p64(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))


@dataclasses.dataclass
class Pairs:
    """Concatenated ASCII sequences with exclusive-prefix offsets (n_pairs + 1 each)."""
    ref: np.ndarray      # uint8
    ref_off: np.ndarray  # uint64
    qry: np.ndarray      # uint8
    qry_off: np.ndarray  # uint64

    @property
    def n_pairs(self) -> int:
        return len(self.ref_off) - 1

    def pair(self, p: int):
        r = self.ref[self.ref_off[p]:self.ref_off[p + 1]].tobytes()
        q = self.qry[self.qry_off[p]:self.qry_off[p + 1]].tobytes()
        return r, q

    def subset(self, idx) -> "Pairs":
        return from_list([self.pair(int(p)) for p in idx])


def lengths(cfg: Config, k0: int = 0, k1: Optional[int] = None):
    k1 = cfg.n_pairs if k1 is None else k1
    n = k1 - k0
    rl = np.zeros(n, np.uint64)
    ql = np.zeros(n, np.uint64)
    c = cfg._c()
    _load().synth_lengths(ctypes.byref(c), cfg.seed, k0, k1, _p64(rl), _p64(ql))
    return rl, ql


def generate(cfg: Config, k0: int = 0, k1: Optional[int] = None, threads: Optional[int] = None,
             pinned_out=None) -> Pairs:
    """Generate pairs [k0, k1) of ``cfg``.  Identical output for any split of the range."""
    k1 = cfg.n_pairs if k1 is None else k1
    rl, ql = lengths(cfg, k0, k1)
    roff = np.zeros(len(rl) + 1, np.uint64)
    qoff = np.zeros(len(ql) + 1, np.uint64)
    np.cumsum(rl, out=roff[1:])
    np.cumsum(ql, out=qoff[1:])
    if pinned_out is not None:
        R, Q = pinned_out(int(roff[-1]), int(qoff[-1]))
    else:
        R = np.empty(int(roff[-1]), np.uint8)
        Q = np.empty(int(qoff[-1]), np.uint8)
    c = cfg._c()
    nt = threads or min(64, os.cpu_count() or 1)
    _load().synth_fill(ctypes.byref(c), cfg.seed, k0, k1, _p64(roff), _p64(qoff),
                       ctypes.c_void_p(R.ctypes.data), ctypes.c_void_p(Q.ctypes.data), nt)
    return Pairs(R, roff, Q, qoff)


def lengths_idx(cfg: Config, idx):
    """(ref, query) lengths of pairs idx[0..] of cfg's stream."""
    idx = np.ascontiguousarray(idx, np.uint64)
    rl = np.zeros(len(idx), np.uint64)
    ql = np.zeros(len(idx), np.uint64)
    c = cfg._c()
    _load().synth_lengths_idx(ctypes.byref(c), cfg.seed, _p64(idx), len(idx), _p64(rl), _p64(ql))
    return rl, ql


def generate_idx(cfg: Config, idx, threads: Optional[int] = None, pinned_out=None) -> Pairs:
    """Generate pairs idx[0], idx[1], ... of ``cfg`` (any subset, in that order): position t
    holds exactly the bytes ``generate`` gives pair idx[t]."""
    idx = np.ascontiguousarray(idx, np.uint64)
    rl, ql = lengths_idx(cfg, idx)
    roff = np.zeros(len(rl) + 1, np.uint64)
    qoff = np.zeros(len(ql) + 1, np.uint64)
    np.cumsum(rl, out=roff[1:])
    np.cumsum(ql, out=qoff[1:])
    if pinned_out is not None:
        R, Q = pinned_out(int(roff[-1]), int(qoff[-1]))
    else:
        R = np.empty(int(roff[-1]), np.uint8)
        Q = np.empty(int(qoff[-1]), np.uint8)
    c = cfg._c()
    nt = threads or min(64, os.cpu_count() or 1)
    _load().synth_fill_idx(ctypes.byref(c), cfg.seed, _p64(idx), len(idx), _p64(roff), _p64(qoff),
                           ctypes.c_void_p(R.ctypes.data), ctypes.c_void_p(Q.ctypes.data), nt)
    return Pairs(R, roff, Q, qoff)


def from_list(pairs) -> Pairs:
    """Build a Pairs batch from a list of (ref, qry) byte/str sequences."""
    rs = [p[0].encode() if isinstance(p[0], str) else bytes(p[0]) for p in pairs]
    qs = [p[1].encode() if isinstance(p[1], str) else bytes(p[1]) for p in pairs]
    roff = np.zeros(len(rs) + 1, np.uint64)
    qoff = np.zeros(len(qs) + 1, np.uint64)
    np.cumsum([len(r) for r in rs], out=roff[1:])
    np.cumsum([len(q) for q in qs], out=qoff[1:])
    R = np.frombuffer(b"".join(rs), np.uint8).copy() if rs else np.zeros(0, np.uint8)
    Q = np.frombuffer(b"".join(qs), np.uint8).copy() if qs else np.zeros(0, np.uint8)
    return Pairs(R, roff, Q, qoff)


def random_short_pairs(rng: np.random.Generator, n: int, max_len: int, alphabet: bytes = b"ACGTN",
                       p: Optional[list] = None, related: float = 0.7) -> Pairs:
    """Small random pairs for parity sweeps (tests): a mix of related (mutated) and unrelated."""
    alpha = np.frombuffer(alphabet, np.uint8)
    out = []
    for _ in range(n):
        m = int(rng.integers(1, max_len + 1))
        r = alpha[rng.choice(len(alpha), size=m, p=p)]
        if rng.random() < related:
            q = r.copy()
            mut = rng.random(m) < rng.uniform(0, 0.3)
            q[mut] = alpha[rng.choice(len(alpha), size=int(mut.sum()), p=p)]
            # random indels
            q = list(q)
            for _ in range(int(rng.integers(0, 4))):
                if q and rng.random() < 0.5:
                    del q[int(rng.integers(0, len(q)))]
                else:
                    q.insert(int(rng.integers(0, len(q) + 1)), int(alpha[rng.integers(0, len(alpha))]))
            q = np.array(q if q else [alpha[0]], np.uint8)
            q = q[: int(rng.integers(1, len(q) + 1))] if rng.random() < 0.3 else q
        else:
            nq = int(rng.integers(1, max_len + 1))
            q = alpha[rng.choice(len(alpha), size=nq, p=p)]
        out.append((r.tobytes(), q.tobytes()))
    return from_list(out)
