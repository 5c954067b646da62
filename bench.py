#!/usr/bin/env python
"""Benchmark: GCUPS (and alignments/s) of the guided extension aligner on B200.

Contract (the driver's): ``python bench.py --gpus N --steps K --warmup W`` prints ONE
JSON line on rank 0.  A step is one pass of the whole hot path (SURVEY.md §8(a):
pack, plan, wavefront alignment with Z-drop, result write; for N > 1 plus the NCCL
gather of the result records) over one batch of synthetic pairs of BASELINE.json
configs[1] (C2: 100k HiFi-like pairs of 10-20 kbp, 1% error, band 500, Z-drop 400).

* ``value``      GCUPS of the whole job, inputs resident in HBM when timing starts
                 (cells = the oracle's algorithmic count, bit-checked in parity);
* ``e2e``        the same metric through the public C ABI with pinned HOST buffers:
                 every step copies that step's ASCII inputs in and the result records
                 out inside the timed region;
* ``roofline``   the align kernel's integer-op rate vs the ALU issue peak;
* ``cpu_baseline`` the CPU oracle, as it stands, on a bounded sample of the workload,
                 on the host cores (rank 0 only).

``--impl reference`` times the oracle itself (the reference arm of this tier).
Multi-GPU (torchrun): each rank aligns its own shard of pairs (weak scaling: per-GPU
work fixed), results are gathered with NCCL all_gather; time = max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

# DESIGN.md §6.3 "Roofline": the path is ALU-pipe bound.  Algorithmic work per cell =
# the minimal ALU-pipe lane-instruction count on sm_100a with DPX .S16x2 (two cells per
# lane-instruction) and the Eq. 1 add on the FMA pipe: Eq. 2 0.5 + Eq. 3 0.5 + Eq. 1 0.5
# (3-input max) + S lookup 0.5 + Eq. 5 running max 0.25 = 2.25.  Peak = 148 SMs x 64 ALU lanes/clk (4 SMSP x 16,
# B300_MICROARCH "alu-pipe rt_SMSP=2"; measured 62.4-62.5, profiles/r01_dpx16.jsonl) x
# clocks.max.sm.
OPS_PER_CELL = 2.25
# the same minimal formulation one cell per lane-instruction (the 32-bit kernels)
OPS_PER_CELL_32 = 4.5
SM_COUNT = 148
LANES_PER_CLK_PER_SM = 64
# dram__bytes_read.sum + dram__bytes_write.sum per align launch on the full C2 batch, from
# one ncu capture (profiles/r01c_ncu_align16_dram_c2.csv, r01_ncu_align_kernel_summary.csv);
# updated per profile.
TRAFFIC = {"align_kernel<32>": 1.603e9 + 0.0748e9, "align16_kernel<16>": 3.328e9 + 1.545e9}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--pairs", type=int, default=0, help="pairs per GPU (default: the config's)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=0, help="oracle sample stride (0: auto)")
    ap.add_argument("--order", default="lpt", choices=["lpt", "input"])
    ap.add_argument("--tiers", default="split", choices=["split", "single"],
                    help="16-bit kernel: each pair at its own slot tier (default) or one "
                         "launch at the widest front (ablation; input order implies single)")
    ap.add_argument("--balance", default="static", choices=["static", "dynamic"],
                    help="static: fixed per-rank shards; dynamic: every rank holds the whole "
                         "batch and the persistent kernels claim pairs from one counter in "
                         "rank 0's HBM with system-scope atomics (NEXT #1)")
    return ap.parse_args()


class ClockSampler:
    """NVML SM-clock / throttle-reason sampling during the timed region."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
        "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, device: int):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": [k for k, v in self.REASONS.items() if self.reasons & v and k != "gpu_idle"],
                "samples": len(self.samples)}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_oracle_sample(pairs: synth.Pairs, params: dict, stride: int):
    """The oracle, as it stands, on every `stride`-th pair; returns (idx, results, seconds)."""
    import oracle
    idx = np.arange(0, pairs.n_pairs, stride)
    sub = pairs.subset(idx)
    t0 = time.perf_counter()
    rc, res, _ = oracle.align_batch(sub, params, threads=cpu_cores())
    dt = time.perf_counter() - t0
    assert rc == 0, rc
    return idx, res, dt


def reference_arm(args, cfg, rank, world):
    """--impl reference: the oracle on host cores, each step a bounded sample."""
    if rank != 0:
        return
    n = args.pairs or cfg.n_pairs
    stride = args.cpu_sample or max(1, n // 150)
    pairs = synth.generate(cfg.with_pairs(n))
    params = dict(vars(cfg.scoring))
    for _ in range(args.warmup):
        run_oracle_sample(pairs, params, stride * 4)
    times, cells = [], 0
    for s in range(args.steps):
        idx, res, dt = run_oracle_sample(pairs, params, stride)
        times.append(dt)
        cells += int(res["cells"].sum())
    tot = sum(times)
    value = cells / tot / 1e9
    line = {
        "impl": "reference", "metric": "GCUPS", "value": value, "unit": "GCUPS",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": config_dict(cfg, n, world),
        "cpu_baseline": {"value": value, "unit": "GCUPS", "cores": cpu_cores(), "kind": "oracle",
                         "sample": f"every {stride}th pair of {n} ({len(idx)} pairs per step)"},
        "e2e": {"value": value, "unit": "GCUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_dict(cfg, n_per_gpu, world):
    sc = cfg.scoring
    return {"workload": f"{cfg.name}: {cfg.description}", "pairs_per_gpu": n_per_gpu,
            "global_pairs": n_per_gpu * world, "band": [sc.band_left, sc.band_right],
            "zdrop": sc.zdrop,
            "scoring": {"match": sc.match, "mismatch": sc.mismatch, "ambig": sc.ambig,
                        "gap_open": sc.gap_open, "gap_extend": sc.gap_extend},
            "seed": cfg.seed, "parallelism": f"pairs sharded over {world} GPU(s)",
            "l2": "inputs (GBs of sequence) exceed the 126 MB L2; no flush needed"}


def main():
    args = parse()
    cfg = synth.CONFIGS[args.config]
    rank, world, local = dist_env()
    if args.impl == "reference":
        return reference_arm(args, cfg, rank, world)

    import torch
    import torch.distributed as dist
    from paper_2403_06478_b200 import agatha
    from paper_2403_06478_b200 import dist as adist

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n = args.pairs or cfg.n_pairs
    # rank r aligns pairs [r*n, (r+1)*n) of the config's infinite pair stream (weak scaling)
    full = cfg.with_pairs(n * world)

    # pinned host buffers (used by the e2e leg); inputs copied once to HBM for `value`
    def pinned(nr, nq):
        return (torch.empty(nr, dtype=torch.uint8, pin_memory=True).numpy(),
                torch.empty(nq, dtype=torch.uint8, pin_memory=True).numpy())

    dynamic = args.balance == "dynamic"
    t0 = time.perf_counter()
    # static: rank r holds its shard; dynamic: every rank holds the whole batch (replicated
    # inputs) and claims chunks of it at run time
    k0, k1 = (0, n * world) if dynamic else adist.shard_range(n, rank)
    pairs = synth.generate(full, k0, k1, pinned_out=pinned)
    gen_s = time.perf_counter() - t0
    params = dict(vars(cfg.scoring))
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    d_ref, d_qry = dev(pairs.ref), dev(pairs.qry)
    d_roff, d_qoff = dev(pairs.ref_off.view(np.int64)), dev(pairs.qry_off.view(np.int64))
    n_local = k1 - k0
    d_out = torch.zeros(adist.RECORD_BYTES * n_local, dtype=torch.uint8, device="cuda")
    flags = agatha.ORDER_INPUT if args.order == "input" else 0
    if args.tiers == "single":
        flags |= agatha.SINGLE_TIER
    ctx = agatha.Context(local)
    stream = torch.cuda.current_stream()
    queue = None
    if dynamic:  # NEXT #1: one pair counter in rank 0's HBM, mapped by every rank
        if rank == 0:
            queue = agatha.SharedQueue.create(ctx)
        handle = adist.share_queue_handle(queue.handle if rank == 0 else b"", world)
        if rank != 0:
            queue = agatha.SharedQueue.open(ctx, handle)
    state = {"kernel_ms": 0.0, "launches": 0}

    def start_dynamic():
        if rank == 0:
            queue.reset(stream)
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def step():
        if dynamic:
            start_dynamic()
        agatha.align_batch(ctx, d_ref, d_roff, d_qry, d_qoff, params, out=d_out, flags=flags,
                           stream=stream, queue=queue)
        state["kernel_ms"] = ctx.stats()["align_ms"]
        state["launches"] += ctx.stats()["kernel_launches"]
        if dynamic:
            # cells of the pairs this rank claimed (record word 2 = int64 cells), on device
            state["mine"] = d_out.view(torch.int64).view(-1, 3)[:, 2].sum()
            adist.merge_claimed(d_out, world)  # NCCL all_reduce of the claimed rows
        elif world > 1:
            adist.gather_results(d_out, world)  # NCCL all_gather of the 24-byte records

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    align_ms = []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(stream)
        state["launches"] = 0
        for _ in range(args.steps):
            step()
            align_ms.append(state["kernel_ms"])
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1)
    stats = ctx.stats()
    res = agatha.device_results(d_out)
    ms_max = adist.max_over_ranks(ms, "cuda", world)
    if dynamic:  # res is the merged whole batch; this rank aligned the pairs it claimed
        cells_all = float(res["cells"].sum())
        cells_rank = int(state["mine"].item())
    else:
        cells_rank = int(res["cells"].sum())
        cells_all = adist.sum_over_ranks(float(cells_rank), "cuda", world)
    sec = ms_max / 1e3
    gcups = cells_all * args.steps / sec / 1e9
    aln_s = n * world * args.steps / sec

    # e2e: the public C ABI with pinned host buffers (H2D of inputs + D2H of results each step)
    e2e = None
    if not args.no_e2e:
        host_out = np.zeros(n_local, agatha.RESULT_DTYPE)

        def e2e_step():
            if dynamic:
                start_dynamic()
            agatha.align_batch(ctx, pairs.ref, pairs.ref_off, pairs.qry, pairs.qry_off, params,
                               out=host_out, flags=flags, stream=stream, queue=queue)
            if dynamic and world > 1:  # merge the ranks' claimed rows
                t = torch.from_numpy(host_out.view(np.uint8)).cuda()
                adist.merge_claimed(t, world)
                host_out.view(np.uint8)[:] = t.cpu().numpy()

        e2e_step()
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            e2e_step()
        ev1.record(stream)
        barrier()
        e_ms = adist.max_over_ranks(ev0.elapsed_time(ev1), "cuda", world)
        assert host_out.tobytes() == res.tobytes()
        h2d = int(pairs.ref.nbytes + pairs.qry.nbytes + pairs.ref_off.nbytes + pairs.qry_off.nbytes)
        e2e = {"value": cells_all * args.steps / (e_ms / 1e3) / 1e9, "unit": "GCUPS",
               "alignments_per_s": n * world * args.steps / (e_ms / 1e3),
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 24 * n_local,
               "ms_per_step": e_ms / args.steps}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    # roofline of the dominant kernel (the align kernel), measured live with CUDA events
    align_avg_ms = statistics.mean(align_ms)
    clocks = clk.summary()
    f_ghz = (clocks["sm_max_mhz"] or 1965) / 1e3
    peak_tops = SM_COUNT * LANES_PER_CLK_PER_SM * f_ghz * 1e9 / 1e12
    ops = OPS_PER_CELL if stats.get("packed16") else OPS_PER_CELL_32
    achieved_tops = ops * cells_rank / (align_avg_ms / 1e3) / 1e12
    if stats.get("packed16"):
        tiers = [32 >> t for t in range(3) if stats.get("tier_pairs", [1, 0, 0])[t]]
        kname = " + ".join(f"align16_kernel<{k // 2}>" for k in tiers) or "align16_kernel"
    elif stats.get("warps_per_pair", 1) > 1:
        kname = f"align_wide_kernel<{stats['warps_per_pair']}>"
    else:
        kname = f"align_kernel<{stats['slots_per_lane']}>"
    roofline = {"bound": "alu", "achieved": achieved_tops, "peak": peak_tops,
                "unit": "T ALU lane-instr/s", "frac": achieved_tops / peak_tops,
                "traffic": TRAFFIC.get(kname), "traffic_unit": "bytes/launch (ncu dram read+write)",
                "kernel": kname, "kernel_ms": align_avg_ms,
                "kernel_gcups": cells_rank / (align_avg_ms / 1e3) / 1e9,
                "gcups_roof": peak_tops * 1e12 / ops / 1e9,
                "ops_per_cell": ops,
                "peak_basis": f"148 SM x 64 ALU lanes/clk x {f_ghz:.3f} GHz (clocks.max.sm); "
                              "ops_per_cell = minimal DPX .S16x2 ALU lane-instructions per cell"}

    cpu = None
    parity = None
    if not args.no_cpu:
        # the CPU baseline is timed at N = 1 only; at N > 1 rank 0 still checks a smaller
        # sample of its shard against the oracle (parity), untimed
        stride = args.cpu_sample or max(1, n // (1000 if world == 1 else 200))
        idx, ores, dt = run_oracle_sample(pairs, params, stride)
        if world == 1:
            cpu = {"value": float(ores["cells"].sum()) / dt / 1e9, "unit": "GCUPS", "cores": cpu_cores(),
                   "kind": "oracle", "sample": f"every {stride}th pair of rank 0's {n} ({len(idx)} pairs, "
                                               f"{dt:.1f} s)"}
        mism = int((res[idx] != ores).sum())
        parity = {"pairs_checked": int(len(idx)), "mismatches": mism}

    line = {
        "metric": "GCUPS", "value": gcups, "unit": "GCUPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": dict(config_dict(cfg, n, world), balance=args.balance,
                       parallelism=(f"{world} GPU(s) claim pairs from one shared counter "
                                    "(system-scope atomics, NEXT #1)") if dynamic
                       else f"pairs sharded over {world} GPU(s)"),
        "alignments_per_s": aln_s,
        "cells_per_step": cells_all, "zdrop_terminated": int((res["zdrop_antidiag"] >= 0).sum()),
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": state["launches"],
        "library_launches": stats["library_launches"] * args.steps,
        "stats_last_step": stats, "clocks": clocks, "parity": parity,
        "gen_seconds": gen_s,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
