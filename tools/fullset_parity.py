#!/usr/bin/env python
"""Full-set parity: every pair of a configuration, GPU (through the C ABI, device-resident
inputs as bench.py times them) against the CPU oracle on all host cores, all five result
fields.  One JSON line per configuration.  BASELINE.md plans parity on all pairs for
C2-C5; the oracle costs ~0.9 GCUPS on 16 cores, so this is a one-off run, not a test.

usage (on the GPU box): python tools/fullset_parity.py C3 LS10 C2 > profiles/...jsonl
       python tools/fullset_parity.py --cached C5 C4   (oracle records from
       tools/oracle_cache.py, computed beforehand on the CPU box; only the GPU runs here.
       A config whose cache is incomplete is compared on the chunks that are there.)
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import synth  # noqa: E402


def cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cached_oracle(cfg):
    """(records, mask of pairs covered) from the oracle cache, or (None, None)."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import oracle_cache
    d = oracle_cache.cache_dir(cfg)
    meta_p = os.path.join(d, "meta.json")
    if not os.path.exists(meta_p):
        return None, None
    with open(meta_p) as f:
        chunk = json.load(f)["chunk"]
    exp = np.zeros(cfg.n_pairs, oracle.RESULT_DTYPE)
    have = np.zeros(cfg.n_pairs, bool)
    for k0, k1 in oracle_cache.chunks(cfg.n_pairs, chunk):
        pth = os.path.join(d, f"r_{k0}_{k1}.npy")
        if os.path.exists(pth):
            exp[k0:k1] = np.load(pth)
            have[k0:k1] = True
    return exp, have


def main():
    import torch
    from paper_2403_06478_b200 import agatha

    cached = "--cached" in sys.argv
    names = [a for a in sys.argv[1:] if not a.startswith("--")]
    ctx = agatha.Context(0)
    for name in names:
        cfg = synth.CONFIGS[name]
        pairs = synth.generate(cfg)
        params = vars(cfg.scoring)
        dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
        out = torch.zeros(24 * pairs.n_pairs, dtype=torch.uint8, device="cuda")
        agatha.align_batch(ctx, dev(pairs.ref), dev(pairs.ref_off.view(np.int64)), dev(pairs.qry),
                           dev(pairs.qry_off.view(np.int64)), params, out=out)
        got = agatha.device_results(out)
        stats = ctx.stats()
        if cached:
            exp, have = cached_oracle(cfg)
            if exp is None:
                print(json.dumps({"config": name, "error": "no oracle cache"}), flush=True)
                continue
            dt = None
            got = got[have]
            exp = exp[have]
        else:
            t0 = time.perf_counter()
            rc, exp, _ = oracle.align_batch(pairs, params, threads=cores())
            dt = time.perf_counter() - t0
            assert rc == 0, rc
        diff = {f: int((got[f] != exp[f]).sum()) for f in exp.dtype.names}
        bad = np.nonzero(got != exp)[0]
        line = {"config": name, "pairs": int(pairs.n_pairs), "pairs_compared": int(len(exp)),
                "pairs_differing": int(len(bad)),
                "fields_differing": diff, "cells": int(exp["cells"].sum()),
                "zdrop_terminated": int((exp["zdrop_antidiag"] >= 0).sum()),
                "oracle": "tools/oracle_cache.py (CPU box, computed beforehand)" if cached else "in-run",
                "oracle_seconds": dt, "oracle_cores": None if cached else cores(),
                "oracle_gcups": None if cached else float(exp["cells"].sum()) / dt / 1e9,
                "tier_pairs": stats["tier_pairs"], "packed16": stats["packed16"]}
        if len(bad):
            k = int(bad[0])
            line["first"] = {"pair": k, "gpu": got[k].tolist(), "oracle": exp[k].tolist()}
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
