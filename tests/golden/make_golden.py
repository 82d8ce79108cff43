"""Generate the golden fixtures in tests/golden/ (run in the build container).

Two kinds of fixture:

* ``pinned.json`` -- the known-answer values the reference's own test suite
  pins for the paper's 6x6 GF(3) example and the single-block job cases
  (reference tests/test_jobs.cpp:84-157, tests/test_tasks.cpp:22-372,
  tests/test_chief.cpp:148-236).  Written out here as literals with their
  source lines.
* ``ref_runs.json`` -- outputs of the reference library itself
  (oracle/_ref/libgfrref_ref.so, compiled from /root/reference by
  oracle/Makefile) on seeded small inputs: echelonize block outputs, the
  materialized transformation, single-block ech, mad and the generators.

Usage:  python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402


def M(rows):
    return [list(r) for r in rows]


PINNED = {
    "source": "reference tests (values only)",
    "p": 3,
    # tests/test_tasks.cpp:15-18
    "C00": M([[0, 2, 2], [0, 2, 2], [1, 0, 1]]),
    "C01": M([[0, 1, 0], [1, 2, 2], [0, 2, 1]]),
    "C10": M([[2, 0, 1], [0, 1, 1], [1, 2, 2]]),
    "C11": M([[0, 2, 2], [2, 1, 1], [2, 0, 0]]),
    # tests/test_chief.cpp:22-28
    "C6": M([[0, 2, 2, 0, 1, 0], [0, 2, 2, 1, 2, 2], [1, 0, 1, 0, 2, 1],
             [2, 0, 1, 0, 2, 2], [0, 1, 1, 2, 1, 1], [1, 2, 2, 2, 0, 0]]),
    # tests/test_chief.cpp:148-194 (full blocked output, block 3)
    "C6_out": {
        "rank": 5,
        "upsilon": [[0, 1, 2], [0, 2]],
        "varrho": [[0, 1, 2], [0, 2]],
        "R": {"0,0": [3, 0, []], "0,1": [3, 1, [[0], [0], [1]]], "1,1": [2, 1, [[2], [0]]]},
        "assembled_R": M([[0], [0], [1], [2], [0]]),
        "TM": {"0,0": M([[1, 1, 2], [1, 0, 2], [0, 0, 1]]), "0,1": M([[1, 1], [2, 0], [1, 0]]),
               "1,0": M([[0, 1, 2], [2, 2, 2]]), "1,1": M([[1, 2], [1, 2]])},
        "TK": {"0,0": [0, 3, []], "1,0": [1, 3, [[0, 1, 0]]], "1,1": [1, 2, [[0, 0]]]},
        "T": M([[1, 1, 2, 1, 0, 1], [1, 0, 2, 2, 0, 0], [0, 0, 1, 1, 0, 0],
                [0, 1, 2, 1, 0, 2], [2, 2, 2, 1, 0, 2], [0, 1, 0, 0, 1, 0]]),
        "task_counts": {"ClearDown": 4, "UpdateRow": 2, "UpdateRowTrafo": 6, "Extend": 4,
                        "RowLengthen": 4, "Copy": 2, "PreClearUp": 1, "ClearUp": 3, "total": 26},
        "task_counts_no_transform": {"ClearDown": 4, "UpdateRow": 2, "UpdateRowTrafo": 0, "Extend": 4,
                                     "RowLengthen": 0, "Copy": 2, "PreClearUp": 1, "ClearUp": 1, "total": 14},
    },
    # tests/test_jobs.cpp:84-107
    "mul": [{"b": M([[0, 2], [1, 0]]), "c": M([[0, 1, 0], [0, 2, 1]]), "out": M([[0, 1, 2], [0, 1, 0]])}],
    "mad": [{"a": M([[1], [1], [2]]), "b": M([[2, 0], [0, 1], [1, 2]]), "c": M([[2], [2]]),
             "out": M([[2], [0], [2]])},
            {"a": M([[0, 2, 2], [2, 1, 1], [2, 0, 0]]), "b": M([[2, 0], [0, 1], [1, 2]]),
             "c": M([[0, 1, 2], [0, 1, 0]]), "out": M([[0, 1, 0], [2, 2, 1], [2, 0, 2]])}],
    # tests/test_jobs.cpp:109-157
    "ech": [
        {"h": M([[0, 2, 2], [0, 2, 2], [1, 0, 1]]), "M": M([[0, 2], [1, 0]]), "K": M([[2, 0]]),
         "R": M([[2], [2]]), "rho": [0, 2], "gamma": [0, 1]},
        {"h": M([[1, 0], [0, 1]]), "M": M([[2, 0], [0, 2]]), "K": [], "R": [], "rho": [0, 1], "gamma": [0, 1]},
        {"h": M([[2], [0], [2]]), "M": M([[1]]), "K": M([[0], [2]]), "R": [], "rho": [0], "gamma": [0]},
    ],
    # tests/test_jobs.cpp:212-246 (unh)
    "unh": [{"rho1": [4, [0, 2]], "rho2": [2, [0]], "rho": [0, 1, 2], "u": [0, 1, 0]},
            {"rho1": [3, [0, 1]], "rho2": [1, [0]], "rho": [0, 1, 2], "u": [0, 0, 1]},
            {"rho1": [5, []], "rho2": [5, [1, 4]], "rho": [1, 4], "u": [1, 1]},
            {"rho1": [9, [2, 5, 6]], "rho2": [6, [0, 3, 5]], "rho": [0, 2, 4, 5, 6, 8], "u": [1, 0, 1, 0, 0, 1]}],
    # tests/test_jobs.cpp:265-271 (mkr)
    "mkr": [{"rho1": [3, [0, 2]], "rho2": [3, [0, 1, 2]], "u": [1, 0, 1]},
            {"rho1": [4, [1, 3]], "rho2": [4, [1, 3]], "u": [1, 1]},
            {"rho1": [4, []], "rho2": [4, [0, 3]], "u": [0, 0]}],
    # tests/test_tasks.cpp:22-46, 74-98, 120-184 (task pins on the 6x6 blocks)
    "clear_down_0": {"gamma": [0, 1], "R": M([[2], [2]]), "M": M([[0, 2], [1, 0]]), "K": M([[2, 0]]),
                     "rho_prime": [0, 2]},
    "clear_down_1": {"gamma": [0, 1, 2], "R": [3, 0, []], "A": M([[2, 0], [0, 1], [1, 2]]), "M": M([[1]]),
                     "K": M([[0], [2]]), "rho_prime": [0], "E": M([[2], [2]]), "lambda": [0, 0, 1]},
    "update_row_0": {"B": M([[0, 1, 2], [0, 1, 0]]), "C": M([[1, 1, 2]])},
    "update_row_1": {"B": M([[0, 0, 2], [0, 0, 0], [0, 1, 0]]), "C": M([[2, 2, 1], [2, 2, 2]])},
    "walkthrough": {
        "d1_v0": {"gamma": [0], "R": M([[2, 1]])},
        "m01_first": M([[1, 2, 0]]),
        "m00_v1": M([[0, 1], [1, 2], [0, 1]]),
        "m01": M([[2], [2], [1]]),
        "m10_v1": M([[0, 1, 2], [2, 2, 2]]),
        "k10_v2": M([[0, 1, 0]]),
        "m11": M([[1, 2], [1, 2]]),
        "k11_v2": M([[0, 0]]),
        "m00_len": M([[0, 0, 1], [1, 0, 2], [0, 0, 1]]),
        "m01_len": M([[2, 0], [2, 0], [1, 0]]),
        "r11": M([[2], [0]]),
        "r01": M([[0], [0], [1]]),
        "m00_f": M([[1, 1, 2], [1, 0, 2], [0, 0, 1]]),
        "m01_f": M([[1, 1], [2, 0], [1, 0]]),
    },
}


def ref_run(p, m, n, block, seed, kind="random", inner=None, with_transform=True):
    if kind == "random":
        C = oracle.ref_random_matrix(p, m, n, seed)
    else:
        C = oracle.ref_random_product_matrix(p, m, n, inner, seed)
    out = oracle.ref_echelonize(p, C, block, 1, with_transform)
    a, b = out.a, out.b
    d = {"p": p, "m": m, "n": n, "block": block, "seed": seed, "kind": kind, "inner": inner,
         "with_transform": with_transform, "rank": out.rank,
         "C": C.tolist(),
         "upsilon": [out.upsilon(j).tolist() for j in range(b)],
         "varrho": [out.varrho(i).tolist() for i in range(a)],
         "R": {f"{j},{l}": [*out.block(0, j, l).shape, out.block(0, j, l).tolist()]
               for j in range(b) for l in range(j, b)},
         "assembled_R": out.assembled_R().tolist()}
    if with_transform:
        d["TM"] = {f"{j},{h}": [*out.block(1, j, h).shape, out.block(1, j, h).tolist()]
                   for j in range(b) for h in range(a)}
        d["TK"] = {f"{i},{h}": [*out.block(2, i, h).shape, out.block(2, i, h).tolist()]
                   for i in range(a) for h in range(i + 1)}
        d["T"] = out.materialize_transform().tolist()
    return d


def main():
    assert oracle.ref is not None, "build oracle/_ref first (make -C oracle)"
    with open(os.path.join(HERE, "pinned.json"), "w") as f:
        json.dump(PINNED, f, indent=0)

    runs = []
    cases = [
        (2, 12, 12, 5, 77), (3, 20, 20, 7, 11), (5, 20, 20, 3, 0xB10C), (7, 13, 17, 5, 0x51DE),
        (251, 16, 16, 4, 9), (193, 11, 14, 4, 78), (3, 24, 24, 4, 0x71ED5), (2, 33, 29, 8, 5),
        (3, 29, 41, 13, 6), (251, 37, 29, 8, 7), (2, 40, 40, 40, 8), (7, 9, 31, 4, 12),
    ]
    for p, m, n, blk, seed in cases:
        runs.append(ref_run(p, m, n, blk, seed))
    # low rank / product-form
    for p, m, n, inner, blk, seed in [(2, 24, 24, 6, 5, 3), (7, 30, 22, 10, 8, 4), (251, 20, 26, 7, 6, 5),
                                      (3, 16, 16, 0, 4, 6)]:
        runs.append(ref_run(p, m, n, blk, seed, "product", inner))
    runs.append(ref_run(3, 20, 20, 7, 11, with_transform=False))
    # single-block ech across thresholds
    echs = []
    for p, m, n, seed, thr in [(2, 17, 13, 1, 4), (3, 24, 19, 2, 3), (5, 24, 19, 3, 8), (251, 15, 21, 4, 5),
                               (7, 33, 17, 5, 2), (3, 12, 12, 6, 256)]:
        H = oracle.ref_random_matrix(p, m, n, seed)
        e = oracle.ref_ech(p, H, thr)
        echs.append({"p": p, "H": H.tolist(), "threshold": thr, "rank": e["rank"], "rho": e["rho"].tolist(),
                     "gamma": e["gamma"].tolist(), "M": e["M"].tolist(), "K": e["K"].tolist(),
                     "R": e["R"].tolist(), "m": m, "n": n})
    gens = []
    for p, m, n, seed in [(2, 5, 7, 1), (3, 4, 9, 2), (251, 6, 6, 3), (7, 1, 33, 4)]:
        gens.append({"p": p, "m": m, "n": n, "seed": seed, "kind": "random",
                     "C": oracle.ref_random_matrix(p, m, n, seed).tolist()})
    for p, m, n, inner, seed in [(7, 6, 5, 3, 9), (2, 8, 8, 2, 10)]:
        gens.append({"p": p, "m": m, "n": n, "inner": inner, "seed": seed, "kind": "product",
                     "C": oracle.ref_random_product_matrix(p, m, n, inner, seed).tolist()})
    with open(os.path.join(HERE, "ref_runs.json"), "w") as f:
        json.dump({"source": "oracle/_ref/libgfrref_ref.so (reference compiled from /root/reference)",
                   "echelonize": runs, "ech": echs, "generators": gens}, f)
    print("wrote", len(runs), "echelonize runs,", len(echs), "ech cases,", len(gens), "generator cases")


if __name__ == "__main__":
    main()
