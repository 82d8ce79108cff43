"""GPU tests of the on-device verifier (gfq_verify; reference gfrref::verify,
src/chief.cpp:531-590): valid outputs pass every method, and outputs with a
single corrupted entry, or checked against a different input, fail."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    from paper_1806_04211_b200 import gfrref
    gfrref.lib()
    return gfrref


def bump(G, f, M, r, c):
    """M[r, c] += 1 (mod p) in place, through K1 on raw pointers."""
    one = G.Matrix.from_numpy(np.ones((1, 1), np.uint8))
    ptr, ld = M.device_ptr()
    a, lda = one.device_ptr()
    G.mad_raw(f.p, 1, 1, 1, a, lda, a, lda, ptr + r * ld + c, ld, ptr + r * ld + c, ld)
    G.synchronize()


CASES = [(2, 200, 160, 48, "random"), (3, 150, 150, 40, "product"), (7, 120, 200, 32, "product"),
         (251, 96, 80, 32, "random"), (5, 64, 64, 64, "zero")]


def make(G, f, m, n, kind, seed=3):
    if kind == "random":
        return G.random_matrix(f, m, n, seed)
    if kind == "product":
        return G.random_product_matrix(f, m, n, min(m, n) // 2, seed)
    return G.Matrix.zeros(m, n)


@pytest.mark.parametrize("p,m,n,block,kind", CASES)
@pytest.mark.parametrize("method", ["exact", "freivalds", "auto"])
def test_valid_outputs_pass(G, p, m, n, block, kind, method):
    f = G.FieldSpec(p)
    C = make(G, f, m, n, kind)
    out = G.echelonize(C, f, G.EchelonizeOptions(block=block, threads=2))
    ok, diag, checked = G.verify(C, out, method)
    assert ok, diag
    assert checked == ("exact" if method == "auto" else method)


@pytest.mark.parametrize("p,m,n,block,kind", CASES[:4])
def test_without_transform_row_space(G, p, m, n, block, kind):
    f = G.FieldSpec(p)
    C = make(G, f, m, n, kind)
    out = G.echelonize(C, f, G.EchelonizeOptions(block=block, with_transform=False))
    ok, diag, checked = G.verify(C, out)
    assert ok and checked == "row-space", diag
    # a different input is (almost surely) outside the row space
    C2 = C.numpy()
    C2[0, :] = (C2[0, :] + 1) % p
    if out.rank < min(m, n):
        ok2, diag2, _ = G.verify(C2, out)
        assert not ok2 and "row space" in diag2


@pytest.mark.parametrize("method", ["exact", "freivalds"])
@pytest.mark.parametrize("target", ["TM", "TK", "R", "input"])
def test_corruption_detected(G, method, target):
    p, m, n, block = 3, 160, 140, 40
    f = G.FieldSpec(p)
    C = G.random_product_matrix(f, m, n, 90, 5)
    out = G.echelonize(C, f, G.EchelonizeOptions(block=block, threads=2))
    a, b = out.chop.a(), out.chop.b()
    if target == "TM":
        blk = next(out.block(1, j, h) for j in range(b) for h in range(a) if out.block(1, j, h).rows > 0
                   and out.block(1, j, h).cols > 0)
        bump(G, f, blk, 0, blk.cols - 1)
    elif target == "TK":
        blk = next(out.block(2, i, h) for i in range(a) for h in range(i + 1)
                   if out.block(2, i, h).rows > 0 and out.block(2, i, h).cols > 0)
        bump(G, f, blk, blk.rows - 1, 0)
    elif target == "R":
        blk = next(out.block(0, j, l) for j in range(b) for l in range(j, b)
                   if out.block(0, j, l).rows > 0 and out.block(0, j, l).cols > 0)
        bump(G, f, blk, 0, blk.cols - 1)
    else:
        Cn = C.numpy()
        Cn[m // 2, n // 3] = (Cn[m // 2, n // 3] + 1) % p
        C = G.Matrix.from_numpy(Cn)
    ok, diag, _ = G.verify(C, out, method)
    assert not ok
    assert diag


def test_echelon_shape_violation(G):
    """A nonzero left of a pivot in R is caught by the shape check before
    any product is formed."""
    p = 5
    f = G.FieldSpec(p)
    Cn = G.random_product_matrix(f, 64, 96, 20, 9).numpy()
    Cn[:, 5] = 0  # a non-pivot column left of later pivots
    C = G.Matrix.from_numpy(Cn)
    out = G.echelonize(C, f, G.EchelonizeOptions(block=32))
    ups = out.global_upsilon()
    rest = [c for c in range(96) if c not in set(ups)]
    # R row r, non-pivot column q with rest[q] < ups[r]
    hit = next(((r, q) for r in range(out.rank) for q in range(len(rest)) if rest[q] < ups[r]), None)
    assert hit is not None
    r, q = hit
    # locate the block holding assembled_R[r, q]
    j = next(j for j in range(out.chop.b()) if r < sum(len(out.upsilon[x].members) for x in range(j + 1)))
    r_loc = r - sum(len(out.upsilon[x].members) for x in range(j))
    col, l = q, 0
    while col >= out.chop.col_parts[l] - len(out.upsilon[l].members):
        col -= out.chop.col_parts[l] - len(out.upsilon[l].members)
        l += 1
    bump(G, f, out.block(0, j, l), r_loc, col)
    ok, diag, _ = G.verify(C, out, "freivalds")
    assert not ok and "echelon shape" in diag


def test_verify_sharded_gathered_output(G):
    import threading
    p, m, n, block = 7, 150, 130, 40
    f = G.FieldSpec(p)
    C = G.random_product_matrix(f, m, n, 60, 2)
    comms = G.Comm.loopback(3)
    outs = [None] * 3

    def body(r):
        outs[r] = G.echelonize_dist(comms[r], f, m, n, G.EchelonizeOptions(block=block, threads=2), C=C)

    th = [threading.Thread(target=body, args=(r,)) for r in range(3)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for o in outs:
        for method in ("exact", "freivalds"):
            ok, diag, _ = G.verify(C, o, method)
            assert ok, diag


def test_verify_rejects_incomplete_sharded_output(G):
    import threading
    p, m, n, block = 3, 120, 120, 30
    f = G.FieldSpec(p)
    C = G.random_matrix(f, m, n, 4)
    comms = G.Comm.loopback(2)
    outs = [None] * 2

    def body(r):
        outs[r] = G.echelonize_dist(comms[r], f, m, n, G.EchelonizeOptions(block=block), C=C, gather=False)

    th = [threading.Thread(target=body, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    ok, diag, _ = G.verify(C, outs[0])
    assert not ok and "gather" in diag


def test_verify_agrees_with_oracle_pin(G, pinned):
    """The paper's 6x6 GF(3) example: verify passes and the oracle agrees."""
    p = pinned["p"]
    f = G.FieldSpec(p)
    C = np.array(pinned["C6"], np.uint8)
    out = G.echelonize(C, f, G.EchelonizeOptions(block=3))
    for method in ("exact", "freivalds"):
        ok, diag, _ = G.verify(C, out, method)
        assert ok, diag
    assert out.rank == pinned["C6_out"]["rank"] == oracle.oracle_rref(p, C)["rank"]
