"""GPU parity of the wide fields -- GF(p) with 251 < p < 2^16 and GF(p^k)
with 256 < p^k < 2^20, the rest of the reference's field range
(src/field.cpp:143-149; its chief and acceptance tests use GF(11^3)) --
stored as u32 elements (kernels/wide.cu): generator, contraction, single-
block ECH and the whole Chief, each against the reference library itself
(oracle/_ref, u32 buffers through ref_set_elem_bytes).  Bit-exact."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

# (p, k): prime fields above u8, extension fields above 256 elements
FIELDS = [(257, 1), (65521, 1), (11, 3), (2, 10), (3, 7)]


@pytest.fixture(scope="module")
def G():
    from paper_1806_04211_b200 import gfrref
    gfrref.lib()
    return gfrref


def fields(G, p, k):
    f = G.FieldSpec(p) if k == 1 else G.FieldSpec(p, k)
    rc = p if k == 1 else oracle.ref_ext_code(p, k)
    assert f.wide and f.esize == 4
    return f, rc


@pytest.mark.parametrize("p,k", FIELDS)
def test_wide_generator(G, p, k):
    f, rc = fields(G, p, k)
    for (m, n, seed) in [(7, 9, 1), (64, 33, 2), (1, 1, 3)]:
        np.testing.assert_array_equal(G.random_matrix(f, m, n, seed).numpy(), oracle.ref32_random_matrix(rc, m, n, seed))


@pytest.mark.parametrize("p,k", FIELDS)
def test_wide_mad(G, p, k):
    f, rc = fields(G, p, k)
    for t, (m, kk, n) in enumerate([(7, 5, 9), (40, 70, 33), (1, 1, 1), (65, 130, 31), (3, 0, 4)]):
        a = oracle.ref32_random_matrix(rc, m, kk, 10 * t + 1)
        b = oracle.ref32_random_matrix(rc, kk, n, 10 * t + 2)
        c = oracle.ref32_random_matrix(rc, m, n, 10 * t + 3)
        np.testing.assert_array_equal(G.mad(f, c, a, b).numpy(), oracle.ref32_mad(rc, a, b, c))
        np.testing.assert_array_equal(G.mul(f, a, b).numpy(), oracle.ref32_mad(rc, a, b))


def test_wide_mad_large_sums(G):
    """every entry p-1 over deep K: the prime-field sums stay exact"""
    p = 65521
    f = G.FieldSpec(p)
    for k in (1000, 70000):
        a = np.full((33, k), p - 1, np.uint32)
        b = np.full((k, 40), p - 1, np.uint32)
        want = (k * (p - 1) * (p - 1)) % p
        assert (G.mul(f, a, b).numpy() == want).all()


@pytest.mark.parametrize("p,k", FIELDS)
def test_wide_ech(G, p, k):
    f, rc = fields(G, p, k)
    rng = np.random.default_rng(p + k)
    cases = [oracle.ref32_random_matrix(rc, m, n, 5 + m) for (m, n) in [(7, 5), (5, 7), (64, 64), (100, 130),
                                                                        (130, 100)]]
    low = oracle.ref32_mad(rc, oracle.ref32_random_matrix(rc, 70, 20, 1), oracle.ref32_random_matrix(rc, 20, 90, 2))
    cases.append(low)  # rank 20
    z = oracle.ref32_random_matrix(rc, 50, 60, 9)
    z[:, rng.choice(60, 20, replace=False)] = 0
    z[rng.choice(50, 10, replace=False)] = 0
    cases.append(z)
    for H in cases:
        e = G.ech(f, H)
        w = oracle.ref32_ech(rc, H)
        assert e.rank() == w["rank"]
        assert list(e.rho.members) == list(w["rho"]) and list(e.gamma.members) == list(w["gamma"])
        for key in "MKR":
            np.testing.assert_array_equal(getattr(e, key).numpy(), w[key])


@pytest.mark.parametrize("p,k,m,n,block", [(11, 3, 9, 7, 3), (257, 1, 40, 33, 8), (65521, 1, 50, 50, 16),
                                           (2, 10, 30, 40, 7), (3, 7, 61, 45, 20)])
@pytest.mark.parametrize("with_transform", [True, False])
def test_wide_echelonize_vs_reference(G, p, k, m, n, block, with_transform):
    """block-for-block against gfrref::echelonize; (11, 3, 9, 7, 3) is the
    reference's own chief test case (tests/test_chief.cpp:371)"""
    f, rc = fields(G, p, k)
    C = oracle.ref32_random_matrix(rc, m, n, 2024)
    if p == 257:  # rank-deficient rows
        C[20:30] = oracle.ref32_mad(rc, oracle.ref32_random_matrix(rc, 10, 20, 7), C[:20])
    out = G.echelonize(C, f, G.EchelonizeOptions(block=block, threads=2, with_transform=with_transform))
    want = oracle.ref32_echelonize(rc, C, block, threads=2, with_transform=with_transform)
    assert out.rank == want.rank
    for j in range(want.b):
        assert list(out.upsilon[j].members) == list(want.upsilon(j))
        for l in range(j, want.b):
            np.testing.assert_array_equal(out.block(0, j, l).numpy(), want.block(0, j, l))
    for i in range(want.a):
        assert list(out.varrho[i].members) == list(want.varrho(i))
    if with_transform:
        for j in range(want.b):
            for h in range(want.a):
                np.testing.assert_array_equal(out.block(1, j, h).numpy(), want.block(1, j, h))
        for i in range(want.a):
            for h in range(i + 1):
                np.testing.assert_array_equal(out.block(2, i, h).numpy(), want.block(2, i, h))
        np.testing.assert_array_equal(out.materialize_transform().numpy(), want.materialize_transform())
    np.testing.assert_array_equal(out.assembled_R().numpy(), want.assembled_R())


@pytest.mark.parametrize("p,k", [(257, 1), (11, 3)])
def test_wide_verify(G, p, k):
    """the on-device certificate (exact T.C and Freivalds) on wide fields,
    and its detection of a corrupted input"""
    f, rc = fields(G, p, k)
    C = oracle.ref32_random_matrix(rc, 45, 38, 77)
    C[30:35] = oracle.ref32_mad(rc, oracle.ref32_random_matrix(rc, 5, 30, 8), C[:30])
    out = G.echelonize(C, f, G.EchelonizeOptions(block=10, threads=2))
    for method in ("exact", "freivalds"):
        ok, diag, chk = G.verify(C, out, method)
        assert ok and chk == method, diag
    bad = C.copy()
    bad[3, 4] = (int(bad[3, 4]) + 1) % f.q
    for method in ("exact", "freivalds"):
        ok, diag, _ = G.verify(bad, out, method)
        assert not ok
    ok, diag, chk = G.verify(C, G.echelonize(C, f, G.EchelonizeOptions(block=10, with_transform=False)))
    assert ok and chk == "row-space", diag


def test_wide_gfmat_round_trip(G, tmp_path):
    """GFMAT files of wide fields: the reference writer's bytes and a read
    back to the same device matrix"""
    for f, rc in [fields(G, 65521, 1), fields(G, 3, 7)]:
        C = oracle.ref32_random_matrix(rc, 6, 5, 3)
        path = tmp_path / f"w{f.q}.gfmat"
        G.write_gfmat_file(str(path), f, C)
        f2, M = G.read_gfmat_file(str(path))
        assert f2 == f and M.esize == 4
        np.testing.assert_array_equal(M.numpy(), C)
        text = path.read_text().splitlines()
        assert text[0] == "GFMAT v1" and text[2] == "rows=6 cols=5"
        assert [int(v) for v in text[3].split()] == [int(v) for v in C[0]]
