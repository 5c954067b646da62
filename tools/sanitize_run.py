"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck): both kernels,
the wide-band tier (D > 1024), a two-context shared queue, all three slot tiers (the edge corpus at w = 500 needs all of them), streamed host inputs
in many chunks, the trace path, pack4 and plan on C1 pairs plus an edge corpus."""
import os
import sys

import numpy as np
import torch

os.environ.setdefault("AGATHA_CHUNK_BYTES", "4096")  # many streamed chunks for host inputs

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2403_06478_b200 import agatha  # noqa: E402

# SANITIZE_SMALL=1 (racecheck, which is ~100x slower): fewer pairs and parameter sets, the
# same kernels and paths
SMALL = os.environ.get("SANITIZE_SMALL") == "1"
ctx = agatha.Context(0)
cfg = synth.CONFIGS["C1"]
pairs = synth.generate(cfg, 0, 6 if SMALL else 64)
edge = synth.from_list([("A", "A"), ("ACGT" * 300, "A"), ("A", "ACGT" * 300), ("N" * 50, "N" * 70),
                        ("ACGTTGCA" * 100, "ACGTTGCA" * 99)])
PRMS = (vars(cfg.scoring), dict(vars(cfg.scoring), band_left=500, band_right=500, zdrop=-1),
        dict(vars(cfg.scoring), band_left=504, band_right=504, zdrop=300),
        dict(vars(cfg.scoring), band_left=0, band_right=3),
        dict(vars(cfg.scoring), band_left=0, band_right=0))
for p in (pairs, edge):
    for flags in ((0, agatha.FORCE_32BIT) if SMALL else (0, agatha.FORCE_32BIT, agatha.ORDER_INPUT)):
        for prm in (PRMS[:3] if SMALL else PRMS):
            agatha.align_pairs(ctx, p, prm, flags=flags)
    agatha.align_pairs_ends(ctx, p, PRMS[2])  # the end-score instantiations (NEXT #4)
# wide-band tier (D > 1024: two and four warps per pair, align_wide_kernel)
wide = synth.generate(synth.CONFIGS["CW1"], 0, 3)
wide = synth.from_list([(R[:1800 if SMALL else 3000], Q[:1800 if SMALL else 3000])
                        for R, Q in (wide.pair(k) for k in range(2 if SMALL else 3))])
for prm in (dict(vars(cfg.scoring), band_left=700, band_right=700, zdrop=400),
            dict(vars(cfg.scoring), band_left=1500, band_right=1600, zdrop=-1)):
    agatha.align_pairs(ctx, wide, prm)
# a shared queue (NEXT #1, system-scope claims) drained by two contexts on two threads
import threading  # noqa: E402
ls = synth.generate(synth.CONFIGS["LS10"], 0, 24 if SMALL else 96)
ctx2 = agatha.Context(0)
q = agatha.SharedQueue.create(ctx)
q.reset()
torch.cuda.synchronize()
outs = [np.zeros(ls.n_pairs, agatha.RESULT_DTYPE) for _ in range(2)]
th = [threading.Thread(target=agatha.align_pairs_q, args=(c, ls, vars(synth.CONFIGS["LS10"].scoring), outs[k], q))
      for k, c in enumerate((ctx, ctx2))]
for t in th:
    t.start()
for t in th:
    t.join()
assert int(((outs[0]["cells"] != 0) | (outs[1]["cells"] != 0)).sum()) == ls.n_pairs
q.close()
ctx2.close()
R, Q = pairs.pair(3)
agatha.localmax_trace(ctx, pairs.ref, pairs.ref_off, pairs.qry, pairs.qry_off, vars(cfg.scoring), 3,
                      len(R) + len(Q) + 1)
dev = torch.from_numpy(np.frombuffer(b"ACGTNACGTTTT" * 11, np.uint8).copy()).cuda()
words = torch.zeros((dev.numel() + 7) // 8, dtype=torch.int32, device="cuda")
agatha.pack4(ctx, dev, words, flags=agatha.PACK_REVERSE)
torch.cuda.synchronize()
print("sanitize workload done")
