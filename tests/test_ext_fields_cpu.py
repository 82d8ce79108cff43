"""GF(p^k) (q = p^k <= 256) on CPU: pin the C oracle's extension-field
arithmetic and the product's host FieldSpec against the reference.

* known answers of the reference's own field tests (reference
  tests/test_field.cpp:85-124, in tests/golden/ext_fields.json "known");
* the reference library's add / mul / inv tables, random_matrix, mat_mul_add
  and single-block ech on seeded inputs (tests/golden/make_golden_ext.py);
* live against oracle/_ref when it is built.
No GPU: the product side only uses the host entry points (gfq_field_*).
"""
import json
import os

import numpy as np
import pytest

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def ext():
    with open(os.path.join(HERE, "golden", "ext_fields.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="module")
def G():
    from paper_1806_04211_b200 import gfrref
    return gfrref


def arr(x):
    return np.array(x, np.uint8).reshape(len(x), len(x[0]) if len(x) else 0)


def test_known_answers(ext, G):
    k = ext["known"]
    for p, kk, mod in k["default_modulus"]:
        assert G.default_modulus(p, kk) == mod
    f = G.FieldSpec(3, 2)
    assert f.modulus == (1, 0, 1) and f.order() == 9
    oc = oracle.ext_code(3, 2, [1, 0, 1])
    for a, b, want in k["gf9"]["mul"]:
        assert f.mul(a, b) == want and oracle.field_op(oc, "mul", a, b) == want
    for a, want in k["gf9"]["inv"]:
        assert f.inv(a) == want and oracle.field_op(oc, "inv", a) == want
    for a, b, want in k["gf9"]["add"]:
        assert f.add(a, b) == want and oracle.field_op(oc, "add", a, b) == want
    g = G.FieldSpec(3, 2, k["gf9_explicit"]["modulus"])
    oc2 = oracle.ext_code(3, 2, k["gf9_explicit"]["modulus"])
    for a, b, want in k["gf9_explicit"]["mul"]:
        assert g.mul(a, b) == want and oracle.field_op(oc2, "mul", a, b) == want
    assert g != f and g == G.FieldSpec(3, 2, [2, 1, 1])


def test_field_errors(G):
    with pytest.raises(ValueError, match="not irreducible"):
        G.FieldSpec(3, 2, [1, 1, 1])
    with pytest.raises(ValueError, match="monic of degree k"):
        G.FieldSpec(3, 2, [1, 0, 2])
    with pytest.raises(ValueError, match="p must be prime"):
        G.FieldSpec(4, 2)
    with pytest.raises(ValueError, match="p\\^k must be < 2\\^20"):
        G.FieldSpec(2, 21)
    # reference tests/test_field.cpp:140: characteristic too large
    with pytest.raises(ValueError, match="p must be < 2\\^16"):
        G.FieldSpec(65537)
    # GF(11^3) (q = 1331, u32 storage): the reference's default modulus
    # (tests/test_field.cpp:89)
    assert list(G.FieldSpec(11, 3).modulus) == [4, 1, 0, 1]


@pytest.mark.parametrize("p,k", [(257, 1), (65521, 1), (11, 3), (2, 10), (3, 7), (2, 12)])
def test_wide_field_ops_match_reference(G, p, k):
    """host arithmetic of the wide fields (u32 storage: log / antilog / Zech
    tables for p^k > 256) equals the reference's FieldSpec ops"""
    F = G.FieldSpec(p) if k == 1 else G.FieldSpec(p, k)
    assert F.wide and F.order() == p ** k
    rc = p if k == 1 else oracle.ref_ext_code(p, k)
    rng = np.random.default_rng(p * 31 + k)
    q = p ** k
    for a, b in rng.integers(0, q, (300, 2)):
        a, b = int(a), int(b)
        assert F.add(a, b) == oracle.ref_field_op(rc, "add", a, b)
        assert F.mul(a, b) == oracle.ref_field_op(rc, "mul", a, b)
        assert F.neg(a) == oracle.ref_field_op(rc, "neg", a)
        if a:
            assert F.inv(a) == oracle.ref_field_op(rc, "inv", a)


def test_tables_match_reference(ext, G):
    for f in ext["fields"]:
        p, k, mod, q = f["p"], f["k"], f["modulus"], f["q"]
        F = G.FieldSpec(p, k, mod)
        oc = oracle.ext_code(p, k, mod)
        assert F.order() == q and list(F.modulus) == mod
        assert [F.inv(a) for a in range(1, q)] == f["inv"]
        assert [oracle.field_op(oc, "inv", a) for a in range(1, q)] == f["inv"]
        if "mul" in f:
            for a in range(q):
                assert [F.mul(a, b) for b in range(q)] == f["mul"][a]
                assert [F.add(a, b) for b in range(q)] == f["add"][a]
                assert [oracle.field_op(oc, "mul", a, b) for b in range(q)] == f["mul"][a]
                assert [oracle.field_op(oc, "add", a, b) for b in range(q)] == f["add"][a]
        # axioms on the whole field
        for a in range(1, q):
            assert F.mul(a, F.inv(a)) == 1
            assert F.add(a, F.neg(a)) == 0


def test_oracle_generators_mad_ech_match_reference(ext):
    for f in ext["fields"]:
        oc = oracle.ext_code(f["p"], f["k"], f["modulus"])
        r = f["random"]
        np.testing.assert_array_equal(oracle.random_matrix(oc, r["m"], r["n"], r["seed"]), arr(r["C"]))
        m = f["mad"]
        A, B, C = arr(m["A"]), arr(m["B"]), arr(m["C"])
        np.testing.assert_array_equal(oracle.mad(oc, A, B, C), arr(m["out"]))
        np.testing.assert_array_equal(oracle.mad(oc, A, B), arr(m["mul"]))
        for e in f["ech"]:
            o = oracle.oracle_rref(oc, arr(e["H"]))
            assert o["rank"] == e["rank"]
            assert o["rho"].tolist() == e["rho"] and o["gamma"].tolist() == e["gamma"]
            for key in "MKR":
                want = np.array(e[key], np.uint8).reshape(o[key].shape)
                np.testing.assert_array_equal(o[key], want)


@pytest.mark.skipif(oracle.ref is None, reason="oracle/_ref not built")
def test_oracle_vs_live_reference_more_cases():
    rng = np.random.default_rng(3)
    for (p, k) in [(2, 5), (2, 6), (2, 7), (3, 4), (3, 5), (13, 2), (11, 2)]:
        mod = oracle.ref_default_modulus(p, k)
        oc, rc = oracle.ext_code(p, k, mod), oracle.ref_ext_code(p, k, mod)
        q = p ** k
        for a in rng.integers(0, q, 20):
            for b in rng.integers(0, q, 20):
                assert oracle.field_op(oc, "mul", int(a), int(b)) == oracle.ref_field_op(rc, "mul", int(a), int(b))
                assert oracle.field_op(oc, "add", int(a), int(b)) == oracle.ref_field_op(rc, "add", int(a), int(b))
        H = oracle.ref_random_product_matrix(rc, 21, 18, 9, 11)
        o, e = oracle.oracle_rref(oc, H), oracle.ref_ech(rc, H, 5)
        assert o["rank"] == e["rank"]
        for key in ("rho", "gamma", "M", "K", "R"):
            np.testing.assert_array_equal(o[key], e[key])
