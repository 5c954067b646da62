#!/usr/bin/env python
"""Oracle result cache: the CPU oracle's records for every pair of a configuration,
computed once on the CPU box and reused by full-set GPU parity runs (SURVEY.md §8(d)
"Timing protocol": parity on all pairs against cached oracle results, keyed by the
generator version, config, seed and params; §5 "Checkpoint / resume").

Test infrastructure: only the oracle writes the cache (this script calls ``oracle`` and
the shared input generator ``synth``, nothing from the CUDA path).

Layout: ``cache/oracle/<config>_<key>/r_<k0>_<k1>.npy`` (RESULT_DTYPE records of pairs
[k0, k1)), plus ``meta.json``.  ``key`` hashes synth.GENERATOR_VERSION, the full config
(lengths, error model, seed, n_pairs, scoring) and ORACLE_SEMANTICS.  Chunks are written
atomically, so an interrupted run resumes where it stopped.

usage: python tools/oracle_cache.py C5 C4 [--threads N] [--chunk PAIRS]
       python tools/oracle_cache.py --status C4 C5
"""
from __future__ import annotations

import argparse
import dataclasses
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import synth  # noqa: E402

CACHE = os.path.join(ROOT, "cache", "oracle")
# Bumped by hand when the oracle's result semantics change (a change of readings in
# DESIGN.md §2); additive outputs that leave the 24-byte record unchanged do not bump it.
ORACLE_SEMANTICS = "r1-readings-R1-R18"


def key(cfg: synth.Config) -> str:
    h = hashlib.sha256()
    h.update(synth.GENERATOR_VERSION.encode())
    h.update(json.dumps(dataclasses.asdict(cfg), sort_keys=True).encode())
    h.update(ORACLE_SEMANTICS.encode())
    return h.hexdigest()[:16]


def cache_dir(cfg: synth.Config) -> str:
    return os.path.join(CACHE, f"{cfg.name}_{key(cfg)}")


def chunks(n: int, chunk: int):
    return [(k0, min(n, k0 + chunk)) for k0 in range(0, n, chunk)]


def _chunk_path(d, k0, k1):
    return os.path.join(d, f"r_{k0}_{k1}.npy")


def status(cfg: synth.Config, chunk: int):
    d = cache_dir(cfg)
    have = [c for c in chunks(cfg.n_pairs, chunk) if os.path.exists(_chunk_path(d, *c))]
    return len(have), len(chunks(cfg.n_pairs, chunk))


def load(cfg: synth.Config, k0: int = 0, k1: int | None = None):
    """Cached oracle records of pairs [k0, k1) of cfg, or None if any chunk is missing."""
    d = cache_dir(cfg)
    meta_p = os.path.join(d, "meta.json")
    if not os.path.exists(meta_p):
        return None
    with open(meta_p) as f:
        chunk = json.load(f)["chunk"]
    k1 = cfg.n_pairs if k1 is None else k1
    parts = []
    for c0, c1 in chunks(cfg.n_pairs, chunk):
        if c1 <= k0 or c0 >= k1:
            continue
        p = _chunk_path(d, c0, c1)
        if not os.path.exists(p):
            return None
        a = np.load(p)
        parts.append(a[max(k0, c0) - c0:min(k1, c1) - c0])
    return np.concatenate(parts) if parts else np.zeros(0, oracle.RESULT_DTYPE)


def fill(cfg: synth.Config, threads: int, chunk: int, log=sys.stderr):
    d = cache_dir(cfg)
    os.makedirs(d, exist_ok=True)
    params = vars(cfg.scoring)
    meta = {"config": dataclasses.asdict(cfg), "key": key(cfg), "chunk": chunk,
            "generator": synth.GENERATOR_VERSION,
            "oracle_semantics": ORACLE_SEMANTICS, "threads": threads}
    with open(os.path.join(d, "meta.json"), "w") as f:
        json.dump(meta, f, indent=1)
    tot_cells, tot_s = 0, 0.0
    for k0, k1 in chunks(cfg.n_pairs, chunk):
        p = _chunk_path(d, k0, k1)
        if os.path.exists(p):
            continue
        pairs = synth.generate(cfg, k0, k1)
        t0 = time.perf_counter()
        rc, res, _ = oracle.align_batch(pairs, params, threads=threads)
        dt = time.perf_counter() - t0
        assert rc == 0, rc
        np.save(p + ".tmp.npy", res)
        os.replace(p + ".tmp.npy", p)
        tot_cells += int(res["cells"].sum())
        tot_s += dt
        print(json.dumps({"config": cfg.name, "k0": k0, "k1": k1, "seconds": round(dt, 1),
                          "gcups": float(res["cells"].sum()) / dt / 1e9, "threads": threads}),
              file=log, flush=True)
    return tot_cells, tot_s


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--chunk", type=int, default=25_000)
    ap.add_argument("--status", action="store_true")
    a = ap.parse_args()
    for name in a.configs:
        cfg = synth.CONFIGS[name]
        if a.status:
            have, tot = status(cfg, a.chunk)
            print(f"{name}: {have}/{tot} chunks in {cache_dir(cfg)}")
        else:
            fill(cfg, a.threads, a.chunk)


if __name__ == "__main__":
    main()
