#!/usr/bin/env python
"""Opcode histogram of one kernel from an .ncu-rep, and for chosen opcodes the source lines that execute them
(needs -lineinfo + --import-source on).  This view found the register-queue moves in the AC2 walk.

    python tools/ncu_opcodes.py gpurun_out/x.ncu-rep k_edges [OPCODE ...]
"""
import csv
import os
import subprocess
import sys
from collections import defaultdict


def main():
    rep, kernel = sys.argv[1], sys.argv[2]
    focus = sys.argv[3:]
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda",
                          "--kernel-name", f"regex:{kernel}"], capture_output=True, text=True).stdout
    fname, hdr, line, src = "?", None, 0, ""
    ops = defaultdict(float)
    by_line = defaultdict(lambda: defaultdict(float))
    seen_fn = None
    for r in csv.reader(out.splitlines()):
        if not r:
            continue
        if r[0] == "File Path":
            fname = os.path.basename(r[1])
        elif r[0] == "Function Name":
            if seen_fn is None:
                seen_fn = r[1]
        elif r[0] == "Line No":
            hdr = {h: i for i, h in enumerate(r)}
            ia, isrc, iex = r.index("Address"), r.index("Address") + 1, r.index("Instructions Executed")
        elif hdr and r[0].isdigit():
            line, src = int(r[0]), r[1].strip()
        elif hdr and r[0] == "" and len(r) > iex and r[ia].startswith("0x"):
            t = r[isrc].split()
            op = t[1] if t and t[0].startswith("@") else (t[0] if t else "?")
            op = ".".join(op.split(".")[:2]) if op.startswith("IMAD") else op.split(".")[0]
            try:
                n = float(r[iex])
            except ValueError:
                continue
            ops[op] += n
            by_line[op][(fname, line, src[:80])] += n
    total = sum(ops.values()) or 1
    print(f"kernel {kernel}: {total / 1e6:.1f} M warp instructions (all captured launches)")
    print(" ".join(f"{k}:{100 * v / total:.1f}" for k, v in sorted(ops.items(), key=lambda kv: -kv[1])[:26]))
    for op in focus:
        print(f"-- {op}: {100 * ops.get(op, 0) / total:.1f}% of all instructions")
        for (f, ln, s), n in sorted(by_line[op].items(), key=lambda kv: -kv[1])[:10]:
            print(f"   {100 * n / total:5.2f}%  {f}:{ln}  {s}")


if __name__ == "__main__":
    main()
