#!/usr/bin/env python
"""Randomised parity sweep: batches with random lengths (mixing all slot tiers), random
bands (0 .. 1100 per side, asymmetric, sometimes unbounded), random scoring (inside and
outside the 16-bit guard), random Z (off, 0 .. 500) and random variant bits, GPU through
the C ABI vs the CPU oracle, all five fields of every pair.  One JSON line per batch plus
a summary; exits non-zero on the first mismatch.

usage (on the GPU box): python tools/random_sweep.py [n_batches] [seed]
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


def mutate(rng, s, err):
    out = []
    for ch in s:
        r = rng.random()
        if r < err * 0.4:
            out.append("ACGT"[int(rng.integers(0, 4))])
        elif r < err * 0.7:
            out.append(ch)
            out.append("ACGT"[int(rng.integers(0, 4))])
        elif r < err:
            continue
        else:
            out.append(ch)
    return "".join(out)


def batch(rng, n):
    lst = []
    for _ in range(n):
        kind = rng.integers(0, 4)
        L = int([rng.integers(1, 200), rng.integers(200, 1500), rng.integers(1500, 6000),
                 rng.integers(6000, 20000)][kind])
        R = "".join("ACGTN"[x] if rng.random() > 0.002 else "N" for x in rng.integers(0, 4, L))
        Q = mutate(rng, R[: int(rng.integers(max(1, L // 2), L + 1))], float(rng.choice([0.01, 0.05, 0.12])))
        if rng.random() < 0.3 and len(Q) > 2:  # chimeric tail: Z-drop fires
            cut = int(rng.integers(1, len(Q)))
            Q = Q[:cut] + "".join("ACGT"[x] for x in rng.integers(0, 4, len(Q) - cut))
        if rng.random() < 0.2:  # a long indel
            x = int(rng.integers(0, max(1, len(Q))))
            Q = Q[:x] + Q[x + int(rng.integers(1, 300)):] if rng.random() < 0.5 else \
                Q[:x] + "".join("ACGT"[y] for y in rng.integers(0, 4, int(rng.integers(1, 300)))) + Q[x:]
        lst.append((R, Q or "A"))
    return lst


def params(rng):
    a = int(rng.integers(1, 6)) if rng.random() < 0.8 else int(rng.integers(6, 60))
    b = int(rng.integers(1, 9))
    n = int(rng.integers(0, b + 1))
    ge = int(rng.integers(0, 4))
    go = ge + int(rng.integers(0, 8))
    bl = int(rng.choice([int(rng.integers(0, 64)), int(rng.integers(64, 520)), int(rng.integers(520, 1100)), -1]))
    br = bl if rng.random() < 0.6 else int(rng.choice([int(rng.integers(0, 520)), int(rng.integers(520, 1100)), -1]))
    if (bl < 0 or br < 0) and rng.random() < 0.8:  # unbounded sides only with short pairs below
        bl, br = max(bl, 0), max(br, 0)
    z = int(rng.choice([-1, int(rng.integers(0, 50)), int(rng.integers(50, 500))]))
    var = int(rng.integers(0, 8)) if rng.random() < 0.25 else 0
    return dict(match=a, mismatch=b, ambig=n, gap_open=go, gap_extend=ge, band_left=bl,
                band_right=br, zdrop=z, variant=var)


def exceeds_limits(lst, prm) -> bool:
    """True when at least one pair is outside the GPU's documented range:
    clipped band D > 4096, or alpha + max(bl,br)*beta + max(a,b,n)*min(m,n) >= 2^20 - 16."""
    mx = max(prm["match"], prm["mismatch"], prm.get("ambig", prm["mismatch"]))
    for R, Q in lst:
        m, n = len(R), len(Q)
        bl = n if prm["band_left"] < 0 or prm["band_left"] > n else prm["band_left"]
        br = m if prm["band_right"] < 0 or prm["band_right"] > m else prm["band_right"]
        if bl + br + 1 > 4096:
            return True
        if prm["gap_open"] + max(bl, br) * prm["gap_extend"] + mx * min(m, n) >= (1 << 20) - 16:
            return True
    return False


def main():
    from paper_2403_06478_b200 import agatha
    nb = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 2026
    rng = np.random.default_rng(seed)
    ctx = agatha.Context(0)
    tot_pairs = tot_cells = 0
    t0 = time.time()
    for k in range(nb):
        prm = params(rng)
        lst = batch(rng, int(rng.integers(20, 120)))
        if prm["band_left"] < 0 or prm["band_right"] < 0:
            lst = [(R[:1500], Q[:1500]) for R, Q in lst]  # unbounded: keep the D <= 4096 limit
        pairs = synth.from_list(lst)
        flags = int(rng.choice([0, 0, 0, agatha.ORDER_INPUT, agatha.SINGLE_TIER, agatha.FORCE_32BIT,
                                agatha.STATIC_ASSIGN]))
        want_ends = rng.random() < 0.3  # NEXT #4 end scores on some batches
        gends = None
        try:
            if want_ends:
                got, gends = agatha.align_pairs_ends(ctx, pairs, prm, flags=flags)
            else:
                got = agatha.align_pairs(ctx, pairs, prm, flags=flags)
            rc_gpu = 0
        except agatha.AgathaError as e:
            got, rc_gpu = None, e.code
        rc, exp, eends, _ = oracle.align_batch_ends(pairs, prm)
        st = ctx.stats() if got is not None else {}
        line = {"batch": k, "pairs": pairs.n_pairs, "params": prm, "flags": flags, "rc_gpu": rc_gpu,
                "rc_oracle": rc, "packed16": st.get("packed16"), "tier_pairs": st.get("tier_pairs")}
        if got is None:
            # the GPU may refuse what the oracle accepts only for its documented limits
            # (DESIGN.md §7): some pair must really exceed D <= 4096 or the |H| bound
            line["ok"] = rc_gpu == agatha.ERANGE and exceeds_limits(lst, prm)
            line["limit_checked"] = True
        else:
            bad = np.nonzero(got != exp)[0]
            if gends is not None:
                f5 = ["mqe", "mqe_i", "mte", "mte_j", "end_score"]
                bad_e = np.nonzero(np.any(np.stack([gends[f] != eends[f] for f in f5]), axis=0))[0]
                line["ends_checked"] = True
                line["ends_mismatches"] = int(len(bad_e))
                bad = np.union1d(bad, bad_e)
            line["mismatches"] = int(len(bad))
            line["ok"] = rc == 0 and len(bad) == 0
            if len(bad):
                i = int(bad[0])
                line["first"] = {"pair": i, "m": len(lst[i][0]), "n": len(lst[i][1]),
                                 "gpu": got[i].tolist(), "oracle": exp[i].tolist()}
            tot_pairs += pairs.n_pairs
            tot_cells += int(exp["cells"].sum())
        print(json.dumps(line), flush=True)
        if not line["ok"]:
            sys.exit(1)
    print(json.dumps({"summary": True, "batches": nb, "pairs_compared": tot_pairs, "cells": tot_cells,
                      "seconds": time.time() - t0, "seed": seed}), flush=True)


if __name__ == "__main__":
    main()
