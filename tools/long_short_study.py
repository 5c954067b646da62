#!/usr/bin/env python
"""NEXT #2: the paper's long/short study (§5.6 l.778-795) on B200.

For 1/5/10/25/50% of 4096 bp reads among 128 bp reads (configs LSxx in synth/),
time the alignment with the persistent queue in input order ("original order") and in
longest-first order (the B200 analogue of sorting + uneven bucketing; the queue makes
them one mechanism), and longest-first with every pair at the widest front (no slot
tiers: the 128 bp reads then run in the w=500 front).  Prints one JSON line per (config, order) plus a summary.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(cfg, order, tiers="split"):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", cfg, "--order", order,
                          "--tiers", tiers, "--no-e2e", "--no-cpu", "--steps", "5", "--warmup", "3"],
                         capture_output=True, text=True, cwd=ROOT)
    return json.loads(out.stdout.strip().splitlines()[-1])


def main():
    rows = []
    for pct in (1, 5, 10, 25, 50):
        cfg = f"LS{pct:02d}"
        r = {o: run(cfg, o) for o in ("input", "lpt")}
        r["lpt_single"] = run(cfg, "lpt", "single")
        line = {"config": cfg, "long_pct": pct,
                "gcups_input": r["input"]["value"], "gcups_lpt": r["lpt"]["value"],
                "gcups_lpt_single_tier": r["lpt_single"]["value"],
                "speedup_tiers": r["lpt_single"]["ms_per_step"] / r["lpt"]["ms_per_step"],
                "ms_input": r["input"]["ms_per_step"], "ms_lpt": r["lpt"]["ms_per_step"],
                "speedup_lpt_over_input": r["input"]["ms_per_step"] / r["lpt"]["ms_per_step"],
                "alignments_per_s_lpt": r["lpt"]["alignments_per_s"],
                "kernel_gcups_lpt": r["lpt"]["roofline"]["kernel_gcups"]}
        print(json.dumps(line), flush=True)
        rows.append(line)


if __name__ == "__main__":
    main()
