"""GPU parity of the Chief's composite tasks (reference tests/test_tasks.cpp)
through the C ABI: the pinned 6x6 GF(3) walkthrough and random task chains
against the numpy restatement (oracle/restate.py)."""
import numpy as np
import pytest

import oracle
from oracle import restate as R
from gfq_testutil import arr

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    from paper_1806_04211_b200 import gfrref
    gfrref.lib()
    return gfrref


def test_clear_down_pinned(G, pinned):
    f = G.FieldSpec(3)
    d, a = G.clear_down(f, arr(pinned["C00"]), None, 0)
    c0 = pinned["clear_down_0"]
    assert list(d.gamma.members) == c0["gamma"] and d.R == arr(c0["R"])
    assert a.M == arr(c0["M"]) and a.K == arr(c0["K"]) and list(a.rho_prime.members) == c0["rho_prime"]
    assert a.A is None and a.E is None and a.lam is None
    d0 = G.PkgD(G.mat_build(2, 1, [[2], [2]]), G.IndexSet(3, (0, 1)))
    d1, a1 = G.clear_down(f, arr(pinned["C10"]), d0, 1)
    c1 = pinned["clear_down_1"]
    assert list(d1.gamma.members) == c1["gamma"] and d1.R.shape == (3, 0)
    assert a1.A == arr(c1["A"]) and a1.M == arr(c1["M"]) and a1.K == arr(c1["K"])
    assert a1.E == arr(c1["E"]) and list(a1.lam) == c1["lambda"]
    # zero input -> empty-rank state
    dz, az = G.clear_down(f, np.zeros((3, 4), np.uint8), None, 0)
    assert dz.gamma == G.IndexSet(4, ()) and dz.R.shape == (0, 4) and az.K.shape == (3, 0)
    with pytest.raises(ValueError, match="universe mismatch"):
        G.clear_down(f, arr(pinned["C10"]), G.PkgD(G.Matrix.zeros(1, 3), G.IndexSet(4, (0,))), 1)


def test_update_row_pinned(G, pinned):
    f = G.FieldSpec(3)
    _, a00 = G.clear_down(f, arr(pinned["C00"]), None, 0)
    c1, b0 = G.update_row(f, a00, arr(pinned["C01"]), None, 0)
    assert b0 == arr(pinned["update_row_0"]["B"]) and c1 == arr(pinned["update_row_0"]["C"])
    d0 = G.PkgD(G.mat_build(2, 1, [[2], [2]]), G.IndexSet(3, (0, 1)))
    _, a10 = G.clear_down(f, arr(pinned["C10"]), d0, 1)
    c2, b1 = G.update_row(f, a10, arr(pinned["C11"]), G.mat_build(2, 3, [[0, 1, 2], [0, 1, 0]]), 1)
    assert b1 == arr(pinned["update_row_1"]["B"]) and c2 == arr(pinned["update_row_1"]["C"])
    with pytest.raises(ValueError, match="B must be given iff"):
        G.update_row(f, a00, arr(pinned["C01"]), G.Matrix.zeros(2, 3), 0)
    with pytest.raises(ValueError):
        G.update_row(f, a00, arr(pinned["C01"]), None, 1)


def test_full_walkthrough_pinned(G, pinned):
    """reference tests/test_tasks.cpp:295-372, every intermediate."""
    f = G.FieldSpec(3)
    W = pinned["walkthrough"]
    C00, C01, C10, C11 = (arr(pinned[k]) for k in ("C00", "C01", "C10", "C11"))
    d0_v0, a00 = G.clear_down(f, C00, None, 0)
    e0_v0 = G.extend(a00, None, 0)
    c01_v1, b01_v0 = G.update_row(f, a00, C01, None, 0)
    k00, m00 = G.update_row_trafo(f, a00, None, None, e0_v0, 0, 0, 0)
    d1_v0, a01 = G.clear_down(f, c01_v1, None, 0)
    e0_v1 = G.extend(a01, e0_v0, 1)
    k00, m = G.update_row_trafo(f, a01, k00, None, e0_v1, 0, 0, 1)
    assert m == arr(W["m01_first"]) and k00.shape == (0, 3)
    assert list(d1_v0.gamma.members) == W["d1_v0"]["gamma"] and d1_v0.R == arr(W["d1_v0"]["R"])
    d0_v1, a10 = G.clear_down(f, C10, d0_v0, 1)
    e1_v0 = G.extend(a10, None, 0)
    c11_v1, b01_v1 = G.update_row(f, a10, C11, b01_v0, 1)
    k10, m00_v1 = G.update_row_trafo(f, a10, None, m00, e1_v0, 1, 0, 0)
    k11, m01 = G.update_row_trafo(f, a10, None, None, e1_v0, 1, 1, 0)
    assert m00_v1 == arr(W["m00_v1"]) and m01 == arr(W["m01"])
    d1_v1, a11 = G.clear_down(f, c11_v1, d1_v0, 1)
    e1_v1 = G.extend(a11, e1_v0, 1)
    k10_v2, m10_v1 = G.update_row_trafo(f, a11, k10, G.mat_build(1, 3, [[1, 2, 0]]), e0_v1, 1, 0, 1)
    k11_v2, m11 = G.update_row_trafo(f, a11, k11, None, e1_v1, 1, 1, 1)
    assert m10_v1 == arr(W["m10_v1"]) and k10_v2 == arr(W["k10_v2"])
    assert m11 == arr(W["m11"]) and k11_v2 == arr(W["k11_v2"])
    m00_len = G.row_lengthen(m00_v1, e0_v0, e0_v1)
    m01_len = G.row_lengthen(m01, e1_v0, e1_v1)
    assert m00_len == arr(W["m00_len"]) and m01_len == arr(W["m01_len"])
    r11 = G.copy_d(d1_v1)
    x01, r01_v0 = G.pre_clear_up(b01_v1, d1_v1)
    assert r11 == arr(W["r11"])
    assert G.clear_up(f, r01_v0, x01, r11) == arr(W["r01"])
    assert G.clear_up(f, m00_len, x01, m10_v1) == arr(W["m00_f"])
    assert G.clear_up(f, m01_len, x01, m11) == arr(W["m01_f"])
    assert e0_v1.rho == G.IndexSet(3, (0, 1, 2)) and e1_v1.rho == G.IndexSet(3, (0, 2))


def test_task_argument_rules(G, pinned):
    f = G.FieldSpec(3)
    _, a00 = G.clear_down(f, arr(pinned["C00"]), None, 0)
    e00 = G.PkgE(G.IndexSet(3, (0, 2)), G.BitString((1, 1)))
    with pytest.raises(ValueError, match="h must be <= i"):
        G.update_row_trafo(f, a00, None, None, e00, 0, 1, 0)
    with pytest.raises(ValueError, match="K must be given iff"):
        G.update_row_trafo(f, a00, G.mat_build(1, 2, [[2, 0]]), None, e00, 0, 0, 0)
    with pytest.raises(ValueError, match="M must be given iff"):
        G.update_row_trafo(f, a00, None, G.mat_build(2, 2, [[0, 2], [1, 0]]), e00, 0, 0, 0)
    with pytest.raises(ValueError, match="E must be given iff"):
        G.extend(a00, e00, 0)
    with pytest.raises(ValueError):
        G.row_lengthen(G.mat_build(2, 2, [[1, 2], [1, 2]]), G.PkgE(G.IndexSet(3, (0, 2)), G.BitString((1, 0))),
                       G.PkgE(G.IndexSet(3, (2,)), G.BitString((1,))))


def _d_to_np(d):
    return R.PkgD(d.R.numpy(), R.IndexSet(d.gamma.universe, d.gamma.members))


@pytest.mark.parametrize("p", [2, 3, 251])
def test_random_task_chains_vs_restatement(G, p):
    """Two block rows through ClearDown/UpdateRow/UpdateRowTrafo/Extend,
    each device output compared with the numpy restatement of the
    reference tasks on the same inputs."""
    f = G.FieldSpec(p)
    for seed in range(3):
        alpha, beta = 24 + 8 * seed, 20 + 4 * seed
        low = seed == 2
        top = oracle.random_product_matrix(p, alpha, beta, 5, 40 + seed) if low else \
            oracle.random_matrix(p, alpha, beta, 40 + seed)
        bot = oracle.random_matrix(p, alpha, beta, 60 + seed)
        right0 = oracle.random_matrix(p, alpha, beta + 3, 80 + seed)
        right1 = oracle.random_matrix(p, alpha, beta + 3, 90 + seed)
        gd0, ga0 = G.clear_down(f, top, None, 0)
        rd0, ra0 = R.clear_down(p, top, R.PkgD(), 0)
        assert gd0.R == rd0.R and ga0.M == ra0.M and ga0.K == ra0.K
        gd1, ga1 = G.clear_down(f, bot, gd0, 1)
        rd1, ra1 = R.clear_down(p, bot, rd0, 1)
        assert gd1.R == rd1.R and list(gd1.gamma.members) == list(rd1.gamma.members)
        assert ga1.A == ra1.A and ga1.E == ra1.E and ga1.M == ra1.M and ga1.K == ra1.K
        assert list(ga1.lam) == list(ra1.lam)
        gc0, gb0 = G.update_row(f, ga0, right0, None, 0)
        rc0, rb0 = R.update_row(p, ra0, right0, None, 0)
        assert gc0 == rc0 and gb0 == rb0
        gc1, gb1 = G.update_row(f, ga1, right1, gb0, 1)
        rc1, rb1 = R.update_row(p, ra1, right1, rb0, 1)
        assert gc1 == rc1 and gb1 == rb1
        ge0 = G.extend(ga0, None, 0)
        re0 = R.extend(ra0, None, 0)
        ge1 = G.extend(ga1, None, 0)
        re1 = R.extend(ra1, None, 0)
        assert ge0.rho.members == re0.rho.members and list(ge1.delta) == list(re1.delta)
        gk, gm = G.update_row_trafo(f, ga0, None, None, ge0, 0, 0, 0)
        rk, rm = R.update_row_trafo(p, ra0, None, None, re0, 0, 0, 0)
        assert gk == rk and gm == rm
        gk1, gm1 = G.update_row_trafo(f, ga1, None, gm, ge0, 1, 0, 0)
        rk1, rm1 = R.update_row_trafo(p, ra1, None, rm, re0, 1, 0, 0)
        assert gk1 == rk1 and gm1 == rm1
        gk2, gm2 = G.update_row_trafo(f, ga1, None, None, ge1, 1, 1, 0)
        rk2, rm2 = R.update_row_trafo(p, ra1, None, None, re1, 1, 1, 0)
        assert gk2 == rk2 and gm2 == rm2
        # PreClearUp / ClearUp on the pivotal-row store of the right column
        side = oracle.random_matrix(p, 6, beta + 3, 70 + seed)
        gdr, _ = G.clear_down(f, side, None, 0)
        rdr, _ = R.clear_down(p, side, R.PkgD(), 0)
        x, rr = G.pre_clear_up(gb1, gdr)
        wx, wr = R.pre_clear_up(rb1, rdr)
        assert x == wx and rr == wr
        assert G.clear_up(f, rr, x, gdr.R) == R.clear_up(p, wr, wx, rdr.R)
