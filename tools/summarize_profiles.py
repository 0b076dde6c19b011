#!/usr/bin/env python
"""Turn one profiling round (tools/profile_round.sh <tag>, files under gpurun_out/) into the tracked
summaries under profiles/: bench lines, launch shares, per-kernel ncu summary, source hot spots, and
profiles/traffic.json (DRAM bytes per launch that bench.py reports as roofline.traffic).

    python tools/summarize_profiles.py <tag>
"""
import csv
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

KEYS = [("gpu__time_duration.sum", "gpu__time_duration"), ("dram__bytes_read.sum", "dram_read"),
        ("dram__bytes_write.sum", "dram_write"), ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
        ("launch__registers_per_thread", "regs"), ("smsp__inst_executed.sum", "warp_inst"),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_pct"),
        ("l1tex__t_sector_hit_rate.pct", "l1_hit_pct"), ("lts__t_sector_hit_rate.pct", "l2_hit_pct"),
        ("smsp__thread_inst_executed_per_inst_executed.ratio", "lanes_per_inst"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
        ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "l1_data_pipe_pct"),
        ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall_long_sb"),
        ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall_short_sb"),
        ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall_wait"),
        ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall_barrier")]


def to_bytes(value, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return float(value) * scale


def main():
    tag = sys.argv[1]
    for name in (f"{tag}_bench.json", f"{tag}_bench_reference_arm.json", f"{tag}_launches_bench_1M_a0.csv",
                 f"{tag}_ncu_full_raw.csv"):
        src = os.path.join(OUT, name)
        if os.path.exists(src):
            shutil.copy(src, os.path.join(PROF, name))
    # ---- launch shares
    path = os.path.join(OUT, f"{tag}_launches_bench_1M_a0.csv")
    if os.path.exists(path):
        lines = [l for l in open(path) if l.startswith('"')]
        rows = list(csv.reader(lines))
        hdr = rows[0]
        ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
        ui = hdr.index("Metric Unit")
        acc = defaultdict(list)
        for r in rows[1:]:
            us = float(r[vi].replace(",", "")) * {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(r[ui], 1.0)
            acc[r[ki].split("(")[0]].append(us)
        total = sum(sum(v) for v in acc.values())
        with open(os.path.join(PROF, f"{tag}_launch_shares.txt"), "w") as f:
            f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none, python bench.py --steps 2 --warmup 1; share of summed kernel time\n")
            for k, v in sorted(acc.items(), key=lambda kv: -sum(kv[1])):
                f.write(f"{k[:60]:60s} n={len(v):3d} avg_us={sum(v) / len(v):9.1f} share={100 * sum(v) / total:5.1f}%\n")
    # ---- per-kernel summary + traffic
    path = os.path.join(OUT, f"{tag}_ncu_full_raw.csv")
    traffic, pipes = {}, {}
    if os.path.exists(path):
        rows = list(csv.reader(open(path)))
        hdr, units = rows[0], rows[1]
        ki = hdr.index("Kernel Name")
        seen = set()
        with open(os.path.join(PROF, f"{tag}_ncu_full_summary.txt"), "w") as f:
            f.write("# ncu --set full --clock-control none, tools/one_step.py 1000000 0 (1M atoms, alpha 0), one launch per kernel\n")
            for r in rows[2:]:
                name = r[ki].split("(")[0].replace("void ", "").split("<")[0]
                if name in seen:
                    continue
                seen.add(name)
                parts = []
                for key, short in KEYS:
                    if key in hdr:
                        i = hdr.index(key)
                        parts.append(f"{short}={r[i]}{units[i] if units[i] not in ('', 'inst', 'register/thread') else ''}")
                f.write(f"{name}: " + ", ".join(parts) + "\n")
                i0, i1 = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
                traffic[name] = int(to_bytes(r[i0], units[i0]) + to_bytes(r[i1], units[i1]))

                def val(key):
                    try:
                        return round(float(r[hdr.index(key)].replace(",", "")), 2)
                    except Exception:
                        return None
                # what bench.py reports as roofline.secondary: the pipe / issue view of the kernel
                pipes[name] = {"fp64_pipe_pct": val("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                               "issue_slots_pct": val("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                               "l1_shared_data_pipe_pct": val("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
                               "warps_active_pct": val("sm__warps_active.avg.pct_of_peak_sustained_active"),
                               "registers": val("launch__registers_per_thread"),
                               "warp_instructions": val("smsp__inst_executed.sum")}
        traffic["_note"] = (f"dram__bytes_read.sum + dram__bytes_write.sum per launch (bytes), ncu --set full, bench workload "
                            f"(1M atoms, alpha 0), capture {tag}")
        traffic["_pipes"] = pipes
        json.dump(traffic, open(os.path.join(PROF, "traffic.json"), "w"), indent=1)
    # ---- per-kernel roofline table (alpha 0 from <tag>_ncu_full_raw.csv, alpha 1.4 from <tag>_a14_ncu_full_raw.csv)
    peak = 6548.2
    try:
        peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        pass
    sections = [("1M atoms, alpha = 0", os.path.join(OUT, f"{tag}_ncu_full_raw.csv")),
                ("1M atoms, alpha = 1.4", os.path.join(OUT, f"{tag}_a14_ncu_full_raw.csv"))]
    if any(os.path.exists(pth) for _, pth in sections):
        with open(os.path.join(PROF, f"{tag}_kernel_table.txt"), "w") as f:
            f.write("# Per-kernel roofline view (ncu --set full --clock-control none; one launch each; times are cold-cache ncu times)\n")
            f.write(f"# columns: kernel | time us | DRAM MB (read+write) | DRAM GB/s | % of measured {peak:.0f} GB/s | % of nominal 8000 GB/s | "
                    "FP64 pipe % | warps active % | lanes/instr | warp instr (M)\n")
            for title, pth in sections:
                if not os.path.exists(pth):
                    continue
                if pth.endswith("_a14_ncu_full_raw.csv"):
                    shutil.copy(pth, os.path.join(PROF, os.path.basename(pth)))
                rows = list(csv.reader(open(pth)))
                hdr, units = rows[0], rows[1]
                col = {k: hdr.index(k) for k, _ in KEYS if k in hdr}
                ki = hdr.index("Kernel Name")
                f.write(f"## {title}\n")
                seen = set()
                for r in rows[2:]:
                    name = r[ki].split("(")[0].replace("void ", "").replace("axb::", "")
                    if name in seen:
                        continue
                    seen.add(name)
                    ti = col["gpu__time_duration.sum"]
                    us = float(r[ti].replace(",", "")) * {"ns": 1e-3, "us": 1.0, "ms": 1e3, "usecond": 1.0, "nsecond": 1e-3, "msecond": 1e3}.get(units[ti], 1.0)
                    i0, i1 = col["dram__bytes_read.sum"], col["dram__bytes_write.sum"]
                    mb = (to_bytes(r[i0].replace(",", ""), units[i0]) + to_bytes(r[i1].replace(",", ""), units[i1])) / 1e6
                    gbs = mb / us * 1e3
                    num = lambda key: float(r[col[key]].replace(",", ""))
                    f.write(f"{name:34s} | {us:8.1f} | {mb:7.1f} | {gbs:7.1f} | {100 * gbs / peak:5.1f} | {100 * gbs / 8000:5.1f} | "
                            f"{num('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active'):5.1f} | "
                            f"{num('sm__warps_active.avg.pct_of_peak_sustained_active'):5.1f} | "
                            f"{num('smsp__thread_inst_executed_per_inst_executed.ratio'):5.1f} | {num('smsp__inst_executed.sum') / 1e6:7.1f}\n")
    for name in (f"{tag}_all_configs_one_gpu.jsonl",):
        if os.path.exists(os.path.join(OUT, name)):
            shutil.copy(os.path.join(OUT, name), os.path.join(PROF, name))
    # ---- source hot spots
    rep = os.path.join(OUT, f"{tag}_full.ncu-rep")
    if os.path.exists(rep):
        for k in ("k_edges", "k_tri_tet3", "k_prune_tris", "k_prune_tets"):
            out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_hotspots.py"), rep, k, "14"],
                                 capture_output=True, text=True).stdout
            open(os.path.join(PROF, f"{tag}_hotspots_{k}.txt"), "w").write(out)


if __name__ == "__main__":
    main()
