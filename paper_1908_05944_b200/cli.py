"""Command-line front end wired to the B200 path (reference cli.py:120-278).

    python -m paper_1908_05944_b200 compute --input atoms.xyzr --alpha 0.0 [--output k.txt] [--stats]
    python -m paper_1908_05944_b200 stats   --input k.txt
    python -m paper_1908_05944_b200 bench   --random 100000 --alpha 0.0 [--repeat 3]

Same sub-commands, flags, output formats and exit codes (0 ok, 1 AlphaxError/OSError, 2 ValueError)
as the reference for the part of the surface the hot path serves: XYZR input (array-native, no
``Ball`` objects), ``compute``, ``stats`` and ``bench``.  ``bench`` prints the reference's CSV schema
(``repeat,workers,stage,seconds``: the 8 STAGE_NAMES + total), with the stage seconds taken from the
CUDA events inside the library; ``workers`` is echoed but has no effect (the GPU schedules its own
work).  PDB input and ``validate`` (which needs the exhaustive CPU oracle) are not part of this build.
"""
from __future__ import annotations

import argparse
import sys
import time

from . import synth
from .errors import AlphaxError
from .io import parse_xyzr_arrays, read_complex, stats_csv, write_complex
from .pipeline import STAGE_NAMES, PipelineConfig, compute_alpha_complex_arrays


def _parse_radius_range(text):
    try:
        lo, hi = (float(p) for p in text.split(":"))
    except ValueError:
        raise ValueError(f"--radius-range must look like LO:HI, got {text!r}") from None
    return lo, hi


def _load(args):
    if getattr(args, "random", None) is not None:
        return synth.random_globule(args.random, seed=args.seed, min_sep=args.min_sep,
                                    radius_range=_parse_radius_range(args.radius_range), density=args.density)
    if args.input is None:
        raise ValueError("an --input file or --random N is required")
    fmt = args.format or ("pdb" if str(args.input).lower().endswith((".pdb", ".ent")) else "xyzr")
    if fmt != "xyzr":
        raise ValueError("only the xyzr input format is part of the B200 build")
    with open(args.input, "r", encoding="utf-8") as handle:
        return parse_xyzr_arrays(handle.read())


def _config(args):
    return PipelineConfig(alpha=args.alpha, mode="grid", chunk_size=getattr(args, "chunk_size", None),
                          workers=1, biomolecule_mode=getattr(args, "biomolecule", False))


def cmd_compute(args) -> int:
    centers, radii = _load(args)
    k = compute_alpha_complex_arrays(centers, radii, _config(args))
    document = write_complex(k)
    if args.output:
        with open(args.output, "w", encoding="utf-8") as handle:
            handle.write(document)
    else:
        sys.stdout.write(document)
    if args.stats:
        sys.stderr.write(stats_csv(k))
    return 0


def cmd_stats(args) -> int:
    with open(args.input, "r", encoding="utf-8") as handle:
        k = read_complex(handle.read())
    sys.stdout.write(stats_csv(k))
    return 0


def cmd_bench(args) -> int:
    centers, radii = _load(args)
    workers_list = [int(w) for w in str(args.workers).split(",")]
    print("repeat,workers,stage,seconds")
    for repeat in range(args.repeat):
        for workers in workers_list:
            times: dict = {}
            start = time.perf_counter()
            k = compute_alpha_complex_arrays(centers, radii, _config(args), stage_times=times)
            io_start = time.perf_counter()
            write_complex(k)
            times["io"] = time.perf_counter() - io_start
            total = time.perf_counter() - start
            # the tiny vertex step has no category of its own (reference cli.py:210); canonical sort +
            # export are this build's share of the reference's merge, reported with the last prune level
            times["prune_edges"] = (times.get("prune_edges", 0.0) + times.pop("prune_vertices", 0.0)
                                    + times.pop("canonical", 0.0) + times.pop("export", 0.0))
            for stage in STAGE_NAMES:
                print(f"{repeat},{workers},{stage},{times.get(stage, 0.0):.6f}")
            print(f"{repeat},{workers},total,{total:.6f}")
    return 0


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="alphax-b200",
                                     description="Alpha complexes of weighted points in 3D on a B200, computed directly "
                                                 "(no Delaunay triangulation). Alpha is given in power-distance units "
                                                 "(squared angstroms).")
    sub = parser.add_subparsers(dest="command", required=True)

    def input_flags(p, required):
        p.add_argument("--input", required=required, help="input file (xyzr)")
        p.add_argument("--format", choices=("xyzr", "pdb"), default=None)

    def random_flags(p):
        p.add_argument("--random", type=int, default=None, metavar="N")
        p.add_argument("--seed", type=int, default=0)
        p.add_argument("--min-sep", type=float, default=1.0)
        p.add_argument("--radius-range", default="1.0:2.0", metavar="LO:HI")
        p.add_argument("--density", type=float, default=0.05)

    c = sub.add_parser("compute", help="compute an alpha complex and write it out")
    input_flags(c, True)
    c.add_argument("--alpha", type=float, required=True)
    c.add_argument("--output", default=None)
    c.add_argument("--chunk-size", type=int, default=None, help="accepted and ignored")
    c.add_argument("--workers", type=int, default=None, help="accepted and ignored")
    c.add_argument("--biomolecule", action="store_true")
    c.add_argument("--stats", action="store_true")
    c.set_defaults(func=cmd_compute)

    s = sub.add_parser("stats", help="print stats for a serialized complex")
    s.add_argument("--input", required=True)
    s.set_defaults(func=cmd_stats)

    b = sub.add_parser("bench", help="per-stage seconds as CSV (CUDA events inside the library)")
    input_flags(b, False)
    random_flags(b)
    b.add_argument("--alpha", type=float, required=True)
    b.add_argument("--repeat", type=int, default=1)
    b.add_argument("--workers", default="1")
    b.add_argument("--chunk-size", type=int, default=None)
    b.add_argument("--biomolecule", action="store_true")
    b.set_defaults(func=cmd_bench)
    return parser


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except AlphaxError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
    except OSError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
    except ValueError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
