#!/usr/bin/env python
"""Per-source-line hot spots of one kernel from an .ncu-rep (needs -lineinfo + --import-source on).

    python tools/ncu_hotspots.py gpurun_out/prof.ncu-rep k_edges [top]
"""
import csv
import os
import subprocess
import sys


def main():
    rep, kernel = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "--kernel-name", f"regex:{kernel}"], capture_output=True, text=True).stdout
    fname, hdr, seen_fn = "?", None, None
    agg = []
    for r in csv.reader(out.splitlines()):
        if not r:
            continue
        if r[0] == "File Path":
            fname = os.path.basename(r[1])
        elif r[0] == "Function Name":
            if seen_fn is None:
                seen_fn = r[1]
            elif r[1] != seen_fn and False:
                break
        elif r[0] == "Line No":
            hdr = {h: i for i, h in enumerate(r)}
        elif r[0].isdigit() and hdr:
            def num(key):
                try:
                    return float(r[hdr[key]])
                except (ValueError, IndexError):
                    return 0.0
            agg.append((fname, int(r[0]), r[1].strip(), num("# Samples"), num("Instructions Executed"),
                        num("Thread Instructions Executed")))
    ts = sum(a[3] for a in agg) or 1
    ti = sum(a[4] for a in agg) or 1
    print(f"kernel {kernel}: {ti:.4g} warp instructions, {ts:.0f} stall samples")
    for f, ln, src, s, i, t in sorted(agg, key=lambda a: -a[3])[:top]:
        print(f"{100 * s / ts:5.1f}% samples {100 * i / ti:5.1f}% inst {t / i if i else 0:5.1f} lanes  {f}:{ln:<4d} {src[:95]}")


if __name__ == "__main__":
    main()
