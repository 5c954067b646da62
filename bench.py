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
Multi-GPU: ``--gpus N`` (N > 1) without a torchrun environment re-launches this script
under ``torch.distributed.run`` with N ranks (one per GPU, 127.0.0.1 rendezvous); with
fewer than N visible GPUs it fails instead of running a smaller job.  The batch is split
by a deterministic LPT partition over nominal cells; ``--scaling weak``
(default: N x the config's pairs, the per-GPU work fixed) or ``strong`` (the config's
fixed batch split N ways, BASELINE.json configs[4]).  Results are gathered with one NCCL
all_gather (shards padded to the largest); time = max over ranks.
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
# SURVEY.md §8(d) roofline: I_cell = 9 int32 lane-instructions per cell (Eq. 1-3 + Eq. 5 on
# sm_100a) against the measured integer lane-instruction rate P_int; the .S16x2 datapath
# the 16-bit kernel runs carries two cells per lane-instruction, so its peak counts two
# int16 lane-ops per lane-instruction (stated in the line).  P_int measured on the B200
# (profiles/r01_int_pipes.jsonl): the highest sustained integer lane-instruction rate of
# the SM, 89.0 lanes/clk/SM (IADD3 at 32 warps/SM, which issues to both the ALU and the
# FMA pipe; an IMNMX + IMAD 1:1 mix reaches 88.1), since the kernel uses both pipes (the
# Eq. 1 add and the selector shifts run on the FMA pipe).  The ALU pipe alone sustains
# 62.4 (VIADDMNMX/VIMNMX3 .S16x2, profiles/r01_dpx16.jsonl): the fraction against that
# is printed too (frac_alu_pipe_only; it exceeds 1 once the kernel needs fewer than
# I_cell / 2 ALU-pipe instructions per cell).
I_CELL = 9
P_INT_LANES_PER_CLK_PER_SM = 89.0
P_ALU_LANES_PER_CLK_PER_SM = 62.4
PAPER_SPEEDUP = {"value": 18.8, "what": "AGAThA vs minimap2 extension (geometric mean over 9 datasets)",
                 "gpu": "NVIDIA RTX A6000", "cpu": "AMD EPYC 7313P 16C/32T, minimap2 SSE4.1",
                 "cite": "PAPER.md l.600-602 (setup), l.673 (18.8x), l.830 (16C32T SSE4)",
                 "note": "the paper's CPU side is an optimised SIMD aligner, not a plain oracle: "
                         "not comparable like for like with cpu_baseline"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None,
                    help="ranks (one per GPU); default 1, or the torchrun world size")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: N x the config's pairs (per-GPU work fixed); strong: the "
                         "config's batch split over the N ranks")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--pairs", type=int, default=0, help="pairs per GPU (default: the config's)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="collective backend (gloo + --same-device: exercise the N-rank path "
                         "on one GPU, for testing)")
    ap.add_argument("--same-device", action="store_true",
                    help="every rank uses cuda:0 (testing the rank logic on a one-GPU box)")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the Z-drop-heavy side measurement (C3) added to the default C2 line")
    ap.add_argument("--cpu-sample", type=int, default=0, help="oracle sample stride (0: auto)")
    ap.add_argument("--order", default="lpt", choices=["lpt", "input"])
    ap.add_argument("--tiers", default="split", choices=["split", "single"],
                    help="16-bit kernel: each pair at its own slot tier (default) or one "
                         "launch at the widest front (ablation; input order implies single)")
    ap.add_argument("--refill", default="queue", choices=["queue", "static"],
                    help="queue: persistent warps refill from the work queue (default); "
                         "static: warp u takes order positions u, u+W, ... (no-refill ablation)")
    ap.add_argument("--balance", default="static", choices=["static", "dynamic"],
                    help="static: fixed per-rank shards; dynamic: every rank holds its shard in "
                         "IPC-shared HBM, the persistent kernels of all ranks claim pairs of the "
                         "federated batch from one counter in rank 0's HBM and read a claimed "
                         "pair from its owner over NVLink (NEXT #1)")
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


def launch_ranks(args) -> int:
    """--gpus N > 1 outside torchrun: re-run this script with N ranks on this node (the
    driver's own launch line), after checking that N GPUs are visible."""
    import socket
    import subprocess

    import torch

    have = torch.cuda.device_count()
    if have < args.gpus and not args.same_device:
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {have}",
              file=sys.stderr, flush=True)
        return 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def newest_profile(pattern: str):
    """The newest committed profile matching profiles/<pattern> (round tags sort by name)."""
    import glob

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", pattern)))
    return files[-1] if files else None


def ncu_kernel_metrics(path: str, kernel_substr: str):
    """{metric: value} of the first launch of a kernel in an `ncu --csv` metrics file, or of
    a tools/ncu_summary.py summary (metric,unit,value)."""
    import csv

    out = {}
    with open(path) as f:
        rows = [r for r in csv.reader(f) if r]
    if rows and rows[0][:3] == ["metric", "unit", "value"]:
        for r in rows[1:]:
            if len(r) == 3:
                try:
                    out[r[0]] = float(r[2])
                except ValueError:
                    pass
        return out
    hdr = next((i for i, r in enumerate(rows) if "Metric Name" in r), None)
    if hdr is None:
        return out
    h = rows[hdr]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    first = None
    for r in rows[hdr + 1:]:
        if len(r) < len(h) or kernel_substr not in r[ki]:
            continue
        first = r[ii] if first is None else first
        if r[ii] == first:
            try:
                out[r[mi]] = float(r[vi].replace(",", ""))
            except ValueError:
                pass
    return out


def cpu_info():
    model, smt = None, None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        with open("/sys/devices/system/cpu/smt/active") as f:
            smt = f.read().strip() == "1"
    except OSError:
        pass
    return {"cpu_model": model, "smt": smt, "logical_cpus": os.cpu_count()}


def cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_oracle_sample(pairs: synth.Pairs, params: dict, stride: int, threads: int = 0):
    """The oracle, as it stands, on every `stride`-th pair; returns (idx, results, seconds)."""
    import oracle
    idx = np.arange(0, pairs.n_pairs, stride)
    sub = pairs.subset(idx)
    t0 = time.perf_counter()
    rc, res, _ = oracle.align_batch(sub, params, threads=threads or cpu_cores())
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
        "cpu_baseline": dict({"value": value, "unit": "GCUPS", "cores": cpu_cores(), "kind": "oracle",
                              "sample": f"every {stride}th pair of {n} ({len(idx)} pairs per step)"},
                             **cpu_info()),
        "paper_speedup": PAPER_SPEEDUP,
        "e2e": {"value": value, "unit": "GCUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_dict(cfg, n_per_gpu, world, n_global=None):
    sc = cfg.scoring
    return {"workload": f"{cfg.name}: {cfg.description}", "pairs_per_gpu": n_per_gpu,
            "global_pairs": n_per_gpu * world if n_global is None else n_global,
            "band": [sc.band_left, sc.band_right],
            "zdrop": sc.zdrop,
            "scoring": {"match": sc.match, "mismatch": sc.mismatch, "ambig": sc.ambig,
                        "gap_open": sc.gap_open, "gap_extend": sc.gap_extend},
            "seed": cfg.seed, "parallelism": f"pairs sharded over {world} GPU(s)",
            "l2": "inputs (GBs of sequence) exceed the 126 MB L2; no flush needed"}


def rank_shard(full: synth.Config, world: int, rank: int, pinned_out=None):
    """§8(e): the deterministic LPT partition of the global batch (full.n_pairs pairs of
    the config's stream) over nominal cells; returns (shards, this rank's pairs).  Every
    rank computes the same partition from the pair lengths alone and generates only its
    own pairs (the generator is counter-based)."""
    from paper_2403_06478_b200 import dist as adist

    n_global = full.n_pairs
    if world == 1:
        return [np.arange(n_global, dtype=np.int64)], synth.generate(full, 0, n_global, pinned_out=pinned_out)
    sc = full.scoring
    rl, ql = synth.lengths(full, 0, n_global)
    w = adist.nominal_cells(rl.astype(np.int64), ql.astype(np.int64), sc.band_left, sc.band_right)
    shards = adist.lpt_partition(w, world)
    return shards, synth.generate_idx(full, shards[rank], pinned_out=pinned_out)


def stream_order(gathered, shards, n_global: int):
    """Records all_gathered from the ranks (each shard padded to the largest; a uint8
    tensor, CUDA or CPU) back into stream order on the host."""
    from paper_2403_06478_b200 import dist as adist

    rows = gathered.cpu().numpy().view(np.dtype([("score", "<i4"), ("ref_end", "<i4"), ("query_end", "<i4"),
                                                  ("zdrop_antidiag", "<i4"), ("cells", "<i8")]))
    return adist.scatter_gathered(rows, shards, n_global)


def main():
    args = parse()
    cfg = synth.CONFIGS[args.config]
    rank, world, local = dist_env()
    if args.impl == "reference":  # the oracle on host cores: rank 0 only, no GPUs needed
        return reference_arm(args, cfg, rank, world)
    if "WORLD_SIZE" not in os.environ and (args.gpus or 1) > 1:
        sys.exit(launch_ranks(args))
    if args.gpus is None:
        args.gpus = world
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but the launch has {world} rank(s)", file=sys.stderr)
        sys.exit(2)

    import torch
    import torch.distributed as dist
    from paper_2403_06478_b200 import agatha
    from paper_2403_06478_b200 import dist as adist

    if args.same_device:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        # NCCL's init log shows the communicator's rank count (nRanks) to the driver
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # stdout carries only the JSON line
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    sc = cfg.scoring
    n_cfg = args.pairs or cfg.n_pairs
    n_global = n_cfg * world if args.scaling == "weak" else n_cfg
    full = cfg.with_pairs(n_global)
    dynamic = args.balance == "dynamic"

    # pinned host buffers (used by the e2e leg); inputs copied once to HBM for `value`
    def pinned(nr, nq):
        return (torch.empty(nr, dtype=torch.uint8, pin_memory=True).numpy(),
                torch.empty(nq, dtype=torch.uint8, pin_memory=True).numpy())

    t0 = time.perf_counter()
    # every rank holds only its own shard (the LPT partition); in the dynamic mode the
    # ranks' kernels also claim pairs of the others' shards and read them over NVLink
    shards, pairs = rank_shard(full, world, rank, pinned)
    mine = shards[rank]
    gen_s = time.perf_counter() - t0
    params = dict(vars(sc))
    n_local = pairs.n_pairs
    ctx = agatha.Context(local)
    if dynamic:
        # NEXT #1: the shard lives in IPC-shareable device buffers; every rank maps the
        # others' (agatha_ipc_open) and aligns the federated batch (all shards in rank
        # order) claiming pairs from one counter in rank 0's HBM
        arrays = (pairs.ref, pairs.ref_off.view(np.uint8), pairs.qry, pairs.qry_off.view(np.uint8))
        own_bufs = [agatha.IpcBuffer.alloc(ctx, a.nbytes) for a in arrays]
        for b_, a in zip(own_bufs, arrays):
            b_.copy_from_host(a)
        meta = (n_local, [b_.handle for b_ in own_bufs], [a.nbytes for a in arrays])
        metas = [meta]
        if world > 1:
            metas = [None] * world
            dist.all_gather_object(metas, meta)
        bufs = [own_bufs if r == rank else [agatha.IpcBuffer.open(ctx, h, nb) for h, nb in zip(metas[r][1], metas[r][2])]
                for r in range(world)]
        owners = [(agatha.DevicePtr(bs[0].ptr, bs[0].nbytes), agatha.DevicePtr(bs[1].ptr, metas[r][0] + 1),
                   agatha.DevicePtr(bs[2].ptr, bs[2].nbytes), agatha.DevicePtr(bs[3].ptr, metas[r][0] + 1))
                  for r, bs in enumerate(bufs)]
        fed_order = np.concatenate(shards)  # global row g of the federated batch -> stream pair
        d_out = torch.zeros(adist.RECORD_BYTES * n_global, dtype=torch.uint8, device="cuda")
        d_out_pad = d_out
        pad = n_local
    else:
        dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
        d_ref, d_qry = dev(pairs.ref), dev(pairs.qry)
        d_roff, d_qoff = dev(pairs.ref_off.view(np.int64)), dev(pairs.qry_off.view(np.int64))
        pad = max(len(x) for x in shards)
        d_out_pad = torch.zeros(adist.RECORD_BYTES * pad, dtype=torch.uint8, device="cuda")
        d_out = d_out_pad[:adist.RECORD_BYTES * n_local]
    flags = agatha.ORDER_INPUT if args.order == "input" else 0
    if args.tiers == "single":
        flags |= agatha.SINGLE_TIER
    if args.refill == "static":
        flags |= agatha.STATIC_ASSIGN
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
            agatha.align_federated(ctx, owners, params, d_out, queue=queue, flags=flags, stream=stream)
        else:
            agatha.align_batch(ctx, d_ref, d_roff, d_qry, d_qoff, params, out=d_out, flags=flags,
                               stream=stream, queue=queue)
        state["kernel_ms"] = ctx.stats()["align_ms"]
        state["launches"] += ctx.stats()["kernel_launches"]
        if dynamic:
            # cells of the pairs this rank claimed (record word 2 = int64 cells), on device
            state["mine"] = d_out.view(torch.int64).view(-1, 3)[:, 2].sum()
            adist.merge_claimed(d_out, world)  # NCCL all_reduce of the claimed rows
        elif world > 1:
            state["gathered"] = adist.gather_results(d_out_pad, world)  # NCCL all_gather

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    align_ms = []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    step_ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(stream)
        state["launches"] = 0
        for k in range(args.steps):
            step()
            step_ev[k].record(stream)  # per-step boundaries (median and min)
            align_ms.append(state["kernel_ms"])
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1)
    step_ms = [ev0.elapsed_time(step_ev[0])] + [step_ev[k - 1].elapsed_time(step_ev[k]) for k in range(1, args.steps)]
    stats = ctx.stats()
    res = agatha.device_results(d_out)
    ms_max = adist.max_over_ranks(ms, "cuda", world)
    ms_mean = adist.sum_over_ranks(ms, "cuda", world) / world  # imbalance = max / mean
    if dynamic:  # res is the merged federated batch; this rank aligned the pairs it claimed
        cells_all = float(res["cells"].sum())
        cells_rank = int(state["mine"].item())
        res_all = np.zeros(n_global, res.dtype)
        res_all[fed_order] = res  # stream order
        res = res_all[mine]       # this rank's own pairs (parity sample below)
    else:
        cells_rank = int(res["cells"].sum())
        cells_all = adist.sum_over_ranks(float(cells_rank), "cuda", world)
    if not dynamic and world > 1:
        res_all = stream_order(state["gathered"], shards, n_global)
        assert res_all[mine].tobytes() == res.tobytes()
        assert float(res_all["cells"].sum()) == cells_all
    sec = ms_max / 1e3
    gcups = cells_all * args.steps / sec / 1e9
    aln_s = n_global * args.steps / sec
    launches_rank = state["launches"]
    launches_all = int(adist.sum_over_ranks(float(launches_rank), "cuda", world))

    # e2e: the public C ABI with pinned host buffers: every step copies this rank's ASCII
    # inputs in, aligns, (N > 1) gathers the records over NCCL, and reads the batch's result
    # records back to the host (scattered into stream order at N > 1)
    e2e = None
    if not args.no_e2e:
        host_out = np.zeros(n_local, agatha.RESULT_DTYPE)
        d_e2e_pad = torch.zeros_like(d_out_pad)
        d_e2e = d_e2e_pad[:adist.RECORD_BYTES * n_local]
        box = {}

        def e2e_step():
            if dynamic:
                # this rank's shard H2D into its shared buffers (the other ranks read them),
                # every rank's copy done before any kernel starts (the barrier in start_dynamic)
                for b_, a in zip(own_bufs, arrays):
                    b_.copy_from_host(a, stream=stream)
                stream.synchronize()
                start_dynamic()
                agatha.align_federated(ctx, owners, params, d_e2e_pad, queue=queue, flags=flags, stream=stream)
                adist.merge_claimed(d_e2e_pad, world)
                if rank == 0:
                    rows = d_e2e_pad.cpu().numpy().view(agatha.RESULT_DTYPE)
                    out_ = np.zeros(n_global, rows.dtype)
                    out_[fed_order] = rows
                    box["res"] = out_
            elif world == 1:
                agatha.align_batch(ctx, pairs.ref, pairs.ref_off, pairs.qry, pairs.qry_off, params,
                                   out=host_out, flags=flags, stream=stream)
                box["res"] = host_out
            else:
                agatha.align_batch(ctx, pairs.ref, pairs.ref_off, pairs.qry, pairs.qry_off, params,
                                   out=d_e2e, flags=flags, stream=stream)
                g = adist.gather_results(d_e2e_pad, world)
                if rank == 0:
                    box["res"] = stream_order(g, shards, n_global)

        e2e_step()
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            e2e_step()
        ev1.record(stream)
        barrier()
        e_ms = adist.max_over_ranks(ev0.elapsed_time(ev1), "cuda", world)
        if dynamic:
            if rank == 0:
                assert box["res"].tobytes() == res_all.tobytes()
            d2h = 24 * n_global if rank == 0 else 0
        elif world == 1:
            assert box["res"].tobytes() == res.tobytes()
            d2h = 24 * n_local
        else:
            if rank == 0:
                assert box["res"][mine].tobytes() == res.tobytes()
                assert box["res"].tobytes() == res_all.tobytes()
            d2h = 24 * pad * world if rank == 0 else 0
        h2d = int(pairs.ref.nbytes + pairs.qry.nbytes + pairs.ref_off.nbytes + pairs.qry_off.nbytes)
        h2d_all = int(adist.sum_over_ranks(float(h2d), "cuda", world))
        e2e = {"value": cells_all * args.steps / (e_ms / 1e3) / 1e9, "unit": "GCUPS",
               "alignments_per_s": n_global * args.steps / (e_ms / 1e3),
               "h2d_bytes_per_step": h2d_all, "d2h_bytes_per_step": d2h,
               "ms_per_step": e_ms / args.steps}
        if world > 1:
            e2e["h2d_bytes_per_step_rank0"] = h2d
            e2e["gather"] = "NCCL all_gather of the 24-byte records (shards padded), then D2H on rank 0"

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    # roofline of the dominant kernel (the align kernel), measured live with CUDA events
    align_avg_ms = statistics.mean(align_ms)
    clocks = clk.summary()
    f_ghz = (clocks["sm_max_mhz"] or 1965) / 1e3
    kernel_gcups = cells_rank / (align_avg_ms / 1e3) / 1e9
    packed16 = bool(stats.get("packed16"))
    if packed16:
        tiers = [32 >> t for t in range(3) if stats.get("tier_pairs", [1, 0, 0])[t]]
        kname = " + ".join(f"align16_kernel<{k // 2}>" for k in tiers) or "align16_kernel"
        ksub = f"align16_kernel<{tiers[0] // 2}" if tiers else "align16_kernel"
    elif stats.get("warps_per_pair", 1) > 1:
        kname = ksub = f"align_wide_kernel<{stats['warps_per_pair']}"
        kname += ">"
    else:
        kname = f"align_kernel<{stats['slots_per_lane']}>"
        ksub = f"align_kernel<{stats['slots_per_lane']}"
    # achieved = I_cell int32 lane-ops per cell x cells / kernel time;
    # peak = P_int (measured lane-instructions/s) x 2 for the .S16x2 datapath (two int16
    # lane-ops per lane-instruction), x 1 for the 32-bit kernels
    lanes_per_instr = 2 if packed16 else 1
    peak_tops = SM_COUNT * P_INT_LANES_PER_CLK_PER_SM * lanes_per_instr * f_ghz * 1e9 / 1e12
    peak_alu_tops = SM_COUNT * P_ALU_LANES_PER_CLK_PER_SM * lanes_per_instr * f_ghz * 1e9 / 1e12
    achieved_tops = I_CELL * kernel_gcups * 1e9 / 1e12
    # the builder's tighter roof: the minimal ALU-pipe instruction count of this kernel's
    # formulation, against 64 ALU lanes/clk/SM
    ops = OPS_PER_CELL if packed16 else OPS_PER_CELL_32
    alu_peak = SM_COUNT * LANES_PER_CLK_PER_SM * f_ghz * 1e9 / 1e12
    roofline = {"bound": "alu", "achieved": achieved_tops, "peak": peak_tops,
                "unit": "T int lane-ops/s", "frac": achieved_tops / peak_tops,
                "kernel": kname, "kernel_ms": align_avg_ms, "kernel_gcups": kernel_gcups,
                "basis": (f"SURVEY.md §8(d): I_cell = {I_CELL} int lane-ops per cell; peak = 148 SM x "
                          f"{P_INT_LANES_PER_CLK_PER_SM} integer lane-instr/clk/SM (the SM's highest measured "
                          f"integer rate, ALU + FMA pipes, profiles/r01_int_pipes.jsonl) x "
                          f"{lanes_per_instr} ({'.S16x2: two int16 lane-ops per lane-instruction' if packed16 else 'int32'})"
                          f" x {f_ghz:.3f} GHz (clocks.max.sm)"),
                "gcups_roof": peak_tops * 1e12 / I_CELL / 1e9,
                "frac_alu_pipe_only": achieved_tops / peak_alu_tops,
                "alu_pipe_only_basis": f"the same against the ALU pipe alone, {P_ALU_LANES_PER_CLK_PER_SM} "
                                       "lane-instr/clk/SM (profiles/r01_dpx16.jsonl)",
                "alu_minimum": {"ops_per_cell": ops, "gcups_roof": alu_peak * 1e12 / ops / 1e9,
                                "frac": kernel_gcups * 1e9 * ops / (alu_peak * 1e12),
                                "basis": "minimal ALU-pipe lane-instructions per cell of this kernel's "
                                         "formulation (DESIGN.md §6.3) vs 148 SM x 64 ALU lanes/clk"}}
    # traffic and pipe utilisation from the newest committed ncu captures of this kernel
    # (kernel-specific file names: the 16-bit kernels' captures are *ncu_align16_*, the
    # wide tier's *ncu_align_wide*, the 32-bit one-warp kernel's *ncu_align_kernel*)
    kfile = "align16" if packed16 else ("align_wide" if stats.get("warps_per_pair", 1) > 1 else "align_kernel")
    dram = newest_profile(f"*ncu_{kfile}*dram*.csv")
    if dram:
        m = ncu_kernel_metrics(dram, ksub)
        if "dram__bytes_read.sum" in m:
            roofline["traffic"] = m["dram__bytes_read.sum"] + m.get("dram__bytes_write.sum", 0.0)
            roofline["traffic_source"] = os.path.relpath(dram, ROOT)
            roofline["traffic_unit"] = "bytes/launch (ncu dram__bytes_read.sum + dram__bytes_write.sum)"
    if "traffic" not in roofline:
        roofline["traffic"] = None
    full_sum = newest_profile(f"*ncu_{kfile}*full_summary.csv")
    if full_sum:
        m = ncu_kernel_metrics(full_sum, ksub)
        key = "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"
        if key in m:
            roofline["ncu_alu_pipe_busy_pct"] = m[key]
            roofline["ncu_issue_active_pct"] = m.get("smsp__issue_active.avg.pct_of_peak_sustained_active")
            roofline["ncu_source"] = os.path.relpath(full_sum, ROOT)

    cpu = None
    parity = None
    if not args.no_cpu:
        # the CPU baseline is timed at N = 1 only; at N > 1 rank 0 still checks a smaller
        # sample of its shard against the oracle (parity), untimed
        stride = args.cpu_sample or max(1, n_local // (1000 if world == 1 else 200))
        idx, ores, dt = run_oracle_sample(pairs, params, stride)
        if world == 1:
            # single-core rate on a smaller sample (every 8th pair of the same sample)
            idx1, ores1, dt1 = run_oracle_sample(pairs, params, stride * 8, threads=1)
            cpu = dict({"value": float(ores["cells"].sum()) / dt / 1e9, "unit": "GCUPS", "cores": cpu_cores(),
                        "kind": "oracle", "sample": f"every {stride}th pair of rank 0's {n_local} ({len(idx)} pairs, "
                                                    f"{dt:.1f} s)",
                        "single_core_gcups": float(ores1["cells"].sum()) / dt1 / 1e9,
                        "single_core_sample": f"every {stride * 8}th pair ({len(idx1)} pairs, {dt1:.1f} s, 1 thread)"},
                       **cpu_info())
        mism = int((res[idx] != ores).sum())
        parity = {"pairs_checked": int(len(idx)), "mismatches": mism}

    # C2 never triggers Z-drop (p_chim = 0): the default run also times the Z-drop-heavy
    # C3 batch (50% chimeric; BASELINE.json configs[2]) on the same context, device-resident
    zdrop_side = None
    if (not args.no_extra and world == 1 and args.config == "C2" and not dynamic
            and args.order == "lpt" and args.tiers == "split" and args.refill == "queue"):
        c3 = synth.CONFIGS["C3"]
        p3 = synth.generate(c3)
        prm3 = dict(vars(c3.scoring))
        d3 = [torch.from_numpy(np.ascontiguousarray(a)).cuda()
              for a in (p3.ref, p3.ref_off.view(np.int64), p3.qry, p3.qry_off.view(np.int64))]
        o3 = torch.zeros(adist.RECORD_BYTES * p3.n_pairs, dtype=torch.uint8, device="cuda")
        agatha.align_batch(ctx, d3[0], d3[1], d3[2], d3[3], prm3, out=o3, stream=stream)
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(3):
            agatha.align_batch(ctx, d3[0], d3[1], d3[2], d3[3], prm3, out=o3, stream=stream)
        ev1.record(stream)
        torch.cuda.synchronize()
        r3 = agatha.device_results(o3)
        ms3 = ev0.elapsed_time(ev1) / 3
        zdrop_side = {"config": f"C3: {c3.description}", "pairs": int(p3.n_pairs),
                      "value": float(r3["cells"].sum()) / (ms3 / 1e3) / 1e9, "unit": "GCUPS",
                      "ms_per_step": ms3, "steps": 3, "warmup": 1,
                      "zdrop_terminated": int((r3["zdrop_antidiag"] >= 0).sum())}
        if not args.no_cpu:
            idx3 = np.arange(0, p3.n_pairs, 1000)
            import oracle
            rc3, e3, _ = oracle.align_batch(p3.subset(idx3), prm3, threads=cpu_cores())
            zdrop_side["parity"] = {"pairs_checked": int(len(idx3)), "mismatches": int((r3[idx3] != e3).sum())}
        del d3, o3

    par = (f"{world} GPU(s) claim pairs of the federated batch from one shared counter (system-scope "
           "atomics; a stolen pair read from its owner's HBM over NVLink, NEXT #1)"
           if dynamic else (f"LPT partition over nominal cells into {world} shards, NCCL all_gather"
                            if world > 1 else "1 GPU"))
    line = {
        "metric": "GCUPS", "value": gcups, "unit": "GCUPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None,
        "dtype": "int16x2 (exact under the host guard; int32 results)" if packed16 else "int32",
        "data": "synthetic",
        "config": dict(config_dict(cfg, n_local, world, n_global), balance=args.balance,
                       parallelism=par, scaling=args.scaling, order=args.order, tiers=args.tiers,
                       refill=args.refill),
        "alignments_per_s": aln_s,
        "step_ms": {"median": statistics.median(step_ms), "min": min(step_ms), "max": max(step_ms),
                    "note": "rank 0's per-step device times; value uses the total over all steps"},
        "cells_per_step": cells_all, "zdrop_terminated": int((res["zdrop_antidiag"] >= 0).sum()),
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "zdrop_workload": zdrop_side,
        "paper_speedup": PAPER_SPEEDUP,
        "gpu_launches": launches_all,
        "library_launches": stats["library_launches"] * args.steps * world,
        "stats_last_step": stats, "clocks": clocks, "parity": parity,
        "gen_seconds": gen_s,
    }
    if world > 1:
        line["rank0_pairs"] = n_local
        line["rank_time"] = {"max_ms_per_step": ms_max / args.steps, "mean_ms_per_step": ms_mean / args.steps,
                             "imbalance": ms_max / ms_mean if ms_mean > 0 else None}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
