"""Generate tests/golden/ext_fields.json: GF(p^k) fixtures (run in the build container).

* ``known`` -- the values the reference's own field tests pin
  (reference tests/test_field.cpp:85-124: default moduli, GF(9) arithmetic
  in the x^2+1 basis, an explicit modulus), written out as literals.
* everything else -- outputs of the reference library itself
  (oracle/_ref/libgfrref_ref.so, compiled from /root/reference by
  oracle/Makefile) over FieldSpec(p, k, modulus): the add / mul tables of the
  small fields, random_matrix, mat_mul_add, single-block ech and blocked
  echelonize (block outputs + materialized transform) on seeded inputs.

Elements use the reference encoding sum_i c_i p^i (q <= 256: one byte).

Usage:  python tests/golden/make_golden_ext.py
"""
from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, HERE)

import oracle  # noqa: E402
from make_golden import ref_run  # noqa: E402

FIELDS = [(2, 2), (2, 3), (2, 4), (2, 8), (3, 2), (3, 3), (5, 2), (7, 2)]

KNOWN = {
    # tests/test_field.cpp:85-90
    "default_modulus": [[2, 2, [1, 1, 1]], [2, 3, [1, 1, 0, 1]], [3, 2, [1, 0, 1]],
                        [3, 3, [1, 2, 0, 1]], [11, 3, [4, 1, 0, 1]]],
    # tests/test_field.cpp:92-102: GF(9), element 3 encodes x
    "gf9": {"mul": [[3, 3, 2], [3, 6, 1], [4, 4, 6]], "inv": [[3, 6]], "add": [[4, 5, 6]]},
    # tests/test_field.cpp:117-124: x^2 + x + 2
    "gf9_explicit": {"modulus": [2, 1, 1], "mul": [[3, 3, 7]]},
}


def main():
    assert oracle.ref is not None, "build oracle/_ref first (make -C oracle)"
    out = {"source": "reference library over FieldSpec(p, k, modulus)", "known": KNOWN, "fields": []}
    seed = 500
    for (p, k) in FIELDS:
        mod = oracle.ref_default_modulus(p, k)
        rc = oracle.ref_ext_code(p, k, mod)
        q = p ** k
        f = {"p": p, "k": k, "modulus": mod, "q": q}
        if q <= 16:
            f["mul"] = [[oracle.ref_field_op(rc, "mul", a, b) for b in range(q)] for a in range(q)]
            f["add"] = [[oracle.ref_field_op(rc, "add", a, b) for b in range(q)] for a in range(q)]
        f["inv"] = [oracle.ref_field_op(rc, "inv", a) for a in range(1, q)]
        f["random"] = {"m": 7, "n": 9, "seed": seed,
                       "C": oracle.ref_random_matrix(rc, 7, 9, seed).tolist()}
        A = oracle.ref_random_matrix(rc, 6, 11, seed + 1)
        B = oracle.ref_random_matrix(rc, 11, 5, seed + 2)
        C = oracle.ref_random_matrix(rc, 6, 5, seed + 3)
        f["mad"] = {"A": A.tolist(), "B": B.tolist(), "C": C.tolist(),
                    "out": oracle.ref_mad(rc, A, B, C).tolist(), "mul": oracle.ref_mad(rc, A, B).tolist()}
        ech = []
        for (m, n, inner, thr) in [(13, 10, 13, 4), (15, 19, 6, 256)]:
            H = oracle.ref_random_product_matrix(rc, m, n, inner, seed + 4 + m)
            e = oracle.ref_ech(rc, H, thr)
            ech.append({"H": H.tolist(), "threshold": thr, "rank": e["rank"],
                        "rho": e["rho"].tolist(), "gamma": e["gamma"].tolist(),
                        "M": e["M"].tolist(), "K": e["K"].tolist(), "R": e["R"].tolist()})
        f["ech"] = ech
        runs = []
        for (m, n, block, kind, inner, wt) in [(12, 12, 5, "random", None, True),
                                                (17, 13, 4, "product", 7, True),
                                                (11, 14, 6, "random", None, False)]:
            r = ref_run(rc, m, n, block, seed + 20 + m, kind, inner, wt)
            r["p"], r["k"], r["modulus"] = p, k, mod
            runs.append(r)
        f["echelonize"] = runs
        out["fields"].append(f)
        seed += 100
    with open(os.path.join(HERE, "ext_fields.json"), "w") as fh:
        json.dump(out, fh, separators=(",", ":"))


if __name__ == "__main__":
    main()
