#!/usr/bin/env python
"""NEXT #2: the paper's long/short study (§5.6 l.778-795) and its ordering
ablation (the analogue of P:754-761) on B200.

For 1/5/10/25/50% of 4096 bp reads among 128 bp reads (configs LSxx in synth/), five
arms, each one bench.py run (every line keeps that run's clock record):
  input_static   input order, no refill (warp u takes positions u, u+W, ...): the
                 analogue of the paper's baseline (original order, no subwarp rejoining)
  input_queue    input order, persistent warps refilled from the queue ("+ refill")
  lpt_static     longest-first order, no refill ("sorted, no queue")
  lpt_single     longest-first + queue, every pair at the widest front (no slot tiers)
  lpt            longest-first + queue + slot tiers (the default)
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(cfg, order, tiers="split", refill="queue"):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", cfg, "--order", order,
                          "--tiers", tiers, "--refill", refill, "--no-e2e", "--no-cpu", "--steps", "5",
                          "--warmup", "3"], capture_output=True, text=True, cwd=ROOT)
    return json.loads(out.stdout.strip().splitlines()[-1])


ARMS = {"input_static": ("input", "single", "static"), "input_queue": ("input", "single", "queue"),
        "lpt_static": ("lpt", "single", "static"), "lpt_single": ("lpt", "single", "queue"),
        "lpt": ("lpt", "split", "queue")}


def main():
    for pct in (1, 5, 10, 25, 50):
        cfg = f"LS{pct:02d}"
        r = {name: run(cfg, *a) for name, a in ARMS.items()}
        line = {"config": cfg, "long_pct": pct}
        for name in ARMS:
            line[f"gcups_{name}"] = r[name]["value"]
            line[f"ms_{name}"] = r[name]["ms_per_step"]
        base = r["input_static"]["ms_per_step"]
        line["speedup_vs_input_static"] = {name: base / r[name]["ms_per_step"] for name in ARMS}
        line["alignments_per_s_lpt"] = r["lpt"]["alignments_per_s"]
        line["kernel_gcups_lpt"] = r["lpt"]["roofline"]["kernel_gcups"]
        line["clocks"] = {name: r[name]["clocks"] for name in ARMS}
        line["parity"] = {name: r[name].get("parity") for name in ARMS}
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
