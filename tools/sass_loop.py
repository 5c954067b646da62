#!/usr/bin/env python
"""Hot-path instruction mix of the steady loop of one align16 kernel instantiation.

Follows the loop from its head along the fall-through path, taking the forward branch
after each step's REDUX (the Z-drop fast path skips the rare argmax block), and counts
opcodes by pipe class.  usage: tools/sass_loop.py LIB.so KERNEL_SUBSTRING
"""
import collections
import re
import subprocess
import sys

ALU = ("VIADDMNMX", "VIMNMX", "VIMNMX3", "PRMT", "LOP3", "SHF", "SEL", "ISETP", "PLOP3", "VOTE", "IADD3", "LEA",
       "FLO", "BREV", "POPC", "IMNMX", "VIADD")
FMA = ("IMAD",)


def kernels(lib):
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    cur, body = None, []
    for line in out.split("\n"):
        m = re.search(r"Function : (\S+)", line)
        if m:
            if cur:
                yield cur, body
            cur, body = m.group(1), []
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m and cur:
            body.append((int(m.group(1), 16), m.group(2).strip()))
    if cur:
        yield cur, body


def steady_path(ins):
    idx = {a: i for i, (a, _) in enumerate(ins)}
    loops = []
    for i, (a, t) in enumerate(ins):
        m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\d,\s*)?0x([0-9a-f]+)", t)
        if m and int(m.group(1), 16) < a:
            body = ins[idx[int(m.group(1), 16)]:i + 1]
            nv = sum("VIADDMNMX.S16x2" in x for _, x in body)
            nr = sum("REDUX" in x for _, x in body)
            if nr in (2, 4) and nv >= 32:
                loops.append((len(body), idx[int(m.group(1), 16)], i))
    # the steady loop: the smallest two-REDUX loop with the DP steps
    _, h, e = min(loops)
    path, i, seen_redux = [], h, False
    while i <= e:
        a, t = ins[i]
        path.append(t)
        if "REDUX" in t:
            seen_redux = True
        m = re.match(r"@!P\d BRA 0x([0-9a-f]+)", t)
        if m and seen_redux:
            i, seen_redux = idx[int(m.group(1), 16)], False
            continue
        i += 1
    return path


def main():
    lib, want = sys.argv[1], sys.argv[2]
    for name, ins in kernels(lib):
        if want not in name:
            continue
        path = steady_path(ins)
        ops = collections.Counter(t.split()[0] if not t.startswith("@") else t.split()[1] for t in path)
        base = collections.Counter()
        for op, n in ops.items():
            base[op.split(".")[0]] += n
        alu = sum(n for op, n in base.items() if op in ALU)
        fma = sum(n for op, n in base.items() if op in FMA)
        print(f"{name}\n  instructions {len(path)}  ALU {alu}  FMA {fma}")
        print("  " + ", ".join(f"{k} {v}" for k, v in sorted(ops.items(), key=lambda x: -x[1])))


if __name__ == "__main__":
    main()
