"""Command-line drop-in for the reference's `gfrref ech` / `gfrref rank`
(reference src/cli.cpp:67-161, exit codes include/gfrref/cli.hpp:10-13),
running the B200 path.

  python -m paper_1806_04211_b200.cli ech --in C.gfmat [--out-r R.gfmat]
      [--out-selects S.txt] [--out-t T.txt] [--block 256] [--threads 1]
      [--no-transform] [--ech-threshold 256] [--remainder-first]
  python -m paper_1806_04211_b200.cli rank --in C.gfmat [--block 256] [--threads 1]

Output files are byte-identical to the reference's; stdout prints "rank r".
"""
from __future__ import annotations

import argparse
import sys

EXIT_OK, EXIT_VERIFY_FAILED, EXIT_BAD_INPUT, EXIT_TASK_FAILURE = 0, 1, 2, 3


def _parser():
    ap = argparse.ArgumentParser(prog="gfq")
    sub = ap.add_subparsers(dest="command", required=True)
    for name in ("ech", "rank"):
        c = sub.add_parser(name)
        c.add_argument("--in", dest="in_path", required=True)
        c.add_argument("--block", type=int, default=256)
        c.add_argument("--threads", type=int, default=1)
        c.add_argument("--ech-threshold", type=int, default=256)
        c.add_argument("--remainder-first", action="store_true")
        if name == "ech":
            c.add_argument("--out-r", default="")
            c.add_argument("--out-selects", default="")
            c.add_argument("--out-t", default="")
            c.add_argument("--no-transform", action="store_true")
    return ap


def main(argv=None) -> int:
    try:
        args = _parser().parse_args(argv)
    except SystemExit as e:
        return EXIT_BAD_INPUT if e.code else EXIT_OK
    from . import gfrref as G
    if args.command == "ech" and args.no_transform and args.out_t:
        print("--out-t conflicts with --no-transform", file=sys.stderr)
        return EXIT_BAD_INPUT
    if args.block < 1 or args.threads < 1:
        print("--block and --threads must be >= 1", file=sys.stderr)
        return EXIT_BAD_INPUT
    try:
        f, C = G.read_gfmat_file(args.in_path)
    except (G.GfqError, ValueError, OSError) as e:
        print(str(e), file=sys.stderr)
        return EXIT_BAD_INPUT
    with_t = args.command == "ech" and not args.no_transform
    opts = G.EchelonizeOptions(block=args.block, threads=args.threads, with_transform=with_t,
                               ech_threshold=args.ech_threshold, remainder_first=args.remainder_first)
    try:
        out = G.echelonize(C, f, opts)
    except (G.GfqError, ValueError, ArithmeticError) as e:
        print(f"task failure: {e}", file=sys.stderr)
        return EXIT_TASK_FAILURE
    if args.command == "ech":
        try:
            if args.out_r:
                G.write_gfmat_file(args.out_r, f, out.assembled_R())
            if args.out_selects:
                out.write_selects_file(args.out_selects)
            if args.out_t:
                out.write_transform_file(args.out_t)
        except (G.GfqError, ValueError, OSError) as e:
            print(str(e), file=sys.stderr)
            return EXIT_BAD_INPUT
    print(f"rank {out.rank}")
    return EXIT_OK


if __name__ == "__main__":
    sys.exit(main())
