#!/usr/bin/env python
"""Summarise an ncu report of the align kernel: key metrics + dynamic SASS opcode mix.

usage: python tools/ncu_summary.py report.ncu-rep [cells_in_launch] > summary.txt
"""
import collections
import csv
import io
import re
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second",
        "sass__inst_executed_local_loads",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
        "smsp__warps_eligible.avg.per_cycle_active"]


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    cells = float(sys.argv[2]) if len(sys.argv) > 2 else None
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    h, u, v = rows[0], rows[1], rows[2]
    d = {h[i]: (v[i], u[i]) for i in range(len(h))}
    print("metric,unit,value")
    for k in KEYS:
        if k in d:
            print(f"{k},{d[k][1]},{d[k][0]}")
    src = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    hh = src[1]
    si, ei = hh.index("Source"), hh.index("Instructions Executed")
    byop = collections.Counter()
    tot = 0
    for r in src[2:]:
        try:
            n = int(r[ei])
        except (ValueError, IndexError):
            continue
        op = re.sub(r"^@!?U?P\w+\s+", "", r[si].strip()).split()
        op = op[0] if op else "?"
        byop[op] += n
        tot += n
    print(f"\n# dynamic SASS mix: {tot} warp instructions"
          + (f", {tot * 32 / cells:.2f} thread-instructions per cell" if cells else ""))
    for op, n in byop.most_common(30):
        print(f"{op},{n},{100 * n / tot:.1f}%" + (f",{n * 32 / cells:.3f}/cell" if cells else ""))


if __name__ == "__main__":
    main()
