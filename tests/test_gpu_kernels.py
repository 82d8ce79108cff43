"""GPU parity of the device kernels and jobs against the CPU oracle.

K1 (tcgen05 kind::i8 contraction + SIMT small-K kernel), K3/K4 gathers and
riffles, K2 ECH, K6 generator.  Integer work: bit-exact comparisons.
"""
import numpy as np
import pytest

import oracle
from oracle import restate as R
from gfq_testutil import arr

pytestmark = pytest.mark.gpu

PRIMES = [2, 3, 7, 193, 251]


@pytest.fixture(scope="module")
def G():
    from paper_1806_04211_b200 import gfrref
    gfrref.lib()
    return gfrref


def rnd(p, m, n, seed):
    return oracle.random_matrix(p, m, n, seed)


# ------------------------------------------------------------------ K1
@pytest.mark.parametrize("policy", [1, 2])
@pytest.mark.parametrize("p", PRIMES)
def test_mad_random_and_ragged(G, p, policy):
    G.set_mad_policy(policy)
    try:
        f = G.FieldSpec(p)
        for t, (m, k, n) in enumerate([(7, 5, 9), (128, 128, 256), (129, 257, 255), (500, 499, 1000),
                                       (1, 1, 1), (300, 32, 17), (64, 1024, 512), (256, 100, 513)]):
            a, b, c = rnd(p, m, k, 10 * t + 1), rnd(p, k, n, 10 * t + 2), rnd(p, m, n, 10 * t + 3)
            np.testing.assert_array_equal(G.mad(f, c, a, b).numpy(), oracle.mad(p, a, b, c))
            np.testing.assert_array_equal(G.mul(f, a, b).numpy(), oracle.mad(p, a, b))
    finally:
        G.set_mad_policy(0)


def test_mad_tc_path_is_taken(G):
    G.mad_counters(reset=True)
    G.set_mad_policy(2)
    try:
        f = G.FieldSpec(3)
        a, b = rnd(3, 256, 512, 1), rnd(3, 512, 256, 2)
        np.testing.assert_array_equal(G.mul(f, a, b).numpy(), oracle.mad(3, a, b))
    finally:
        G.set_mad_policy(0)
    simt, tc = G.mad_counters(reset=True)
    assert tc >= 1


def test_mad_degenerate_shapes(G):
    f = G.FieldSpec(3)
    # reference tests/test_matrix.cpp:72-86 and tests/test_jobs.cpp:97-107
    assert G.mul(f, np.zeros((0, 4), np.uint8), np.zeros((4, 3), np.uint8)).shape == (0, 3)
    z = G.mul(f, np.zeros((3, 0), np.uint8), np.zeros((0, 2), np.uint8))
    assert z.shape == (3, 2) and not z.numpy().any()
    a = rnd(3, 2, 5, 9)
    assert G.mad(f, a, np.zeros((2, 3), np.uint8), rnd(3, 3, 5, 10)) == a
    with pytest.raises(ValueError, match="inner dimensions disagree"):
        G.mul(f, np.zeros((2, 3), np.uint8), np.zeros((2, 3), np.uint8))
    with pytest.raises(ValueError, match="addend shape mismatch"):
        G.mad(f, np.zeros((2, 2), np.uint8), np.zeros((2, 3), np.uint8), np.zeros((3, 3), np.uint8))


@pytest.mark.parametrize("p", [251, 193])
def test_mad_accumulator_bound_max_values(G, p):
    """All entries p-1: the s32 accumulation bound (p-1)^2.K plus the
    addend, and the K-chunking above 2^31 / (p-1)^2."""
    G.set_mad_policy(2)
    try:
        f = G.FieldSpec(p)
        for k in (4096, 8192, 36000):
            a = np.full((130, k), p - 1, np.uint8)
            b = np.full((k, 260), p - 1, np.uint8)
            c = np.full((130, 260), p - 1, np.uint8)
            want = (np.int64(p - 1) * (p - 1) * k + (p - 1)) % p
            got = G.mad(f, c, a, b).numpy()
            assert (got == want).all(), (k, np.unique(got))
    finally:
        G.set_mad_policy(0)


def test_mad_pinned(G, pinned):
    f = G.FieldSpec(pinned["p"])
    for c in pinned["mul"]:
        assert G.mul(f, arr(c["b"]), arr(c["c"])) == arr(c["out"])
    for c in pinned["mad"]:
        assert G.mad(f, arr(c["a"]), arr(c["b"]), arr(c["c"])) == arr(c["out"])


def test_mad_raw_unaligned_views(G):
    """Raw pointers with odd offsets / strides route to the SIMT kernel; same values."""
    import torch
    p = 7
    big = torch.from_numpy(rnd(p, 300, 700, 3)).cuda()
    A = big[1:200, 3:403]          # 199 x 400, base not 16B aligned
    Bm = torch.from_numpy(rnd(p, 400, 250, 4)).cuda()
    D = torch.zeros(199, 250, dtype=torch.uint8, device="cuda")
    G.mad_raw(p, 199, 250, 400, A.data_ptr(), big.stride(0), Bm.data_ptr(), 250, 0, 0, D.data_ptr(), 250)
    torch.cuda.synchronize()
    want = oracle.mad(p, A.cpu().numpy(), Bm.cpu().numpy())
    np.testing.assert_array_equal(D.cpu().numpy(), want)


# ------------------------------------------------------------------ K3 / K4 (jobs)
def test_gathers_and_riffles(G):
    h = arr([[2, 0, 1], [0, 1, 1], [1, 2, 2]])
    sel, rest = G.cex(h, G.IndexSet(3, (0, 1)))
    assert sel == arr([[2, 0], [0, 1], [1, 2]]) and rest == arr([[1], [1], [2]])
    ns, nr = G.cex(h, G.IndexSet(3, ()))
    assert ns.shape == (3, 0) and nr == h
    with pytest.raises(ValueError, match="universe mismatch"):
        G.cex(h, G.IndexSet(4, (0,)))
    h2 = arr([[0, 1, 0], [1, 2, 2], [0, 2, 1]])
    s2, r2 = G.rex(h2, G.IndexSet(3, (0, 2)))
    assert s2 == arr([[0, 1, 0], [0, 2, 1]]) and r2 == arr([[1, 2, 2]])
    assert G.rrf((0, 1, 0), arr([[1, 1], [2, 2]]), arr([[0, 0]])) == arr([[1, 1], [0, 0], [2, 2]])
    assert G.crz(arr([[1], [2]]), (1, 0), 2) == arr([[1, 0], [2, 0]])
    assert G.adi(np.zeros((2, 3), np.uint8), (1, 0, 1)) == arr([[1, 0, 0], [0, 0, 1]])
    assert G.adi(arr([[2, 0]]), (0, 1)) == arr([[2, 1]])
    with pytest.raises(ValueError, match="ones count"):
        G.crz(arr([[1, 2, 0], [0, 1, 2]]), (1, 1), 2)
    with pytest.raises(ValueError, match="more marked positions"):
        G.adi(np.zeros((1, 3), np.uint8), (1, 0, 1))
    with pytest.raises(ValueError, match="bit counts"):
        G.rrf((0, 1), np.zeros((2, 2), np.uint8), np.zeros((1, 2), np.uint8))


def test_gathers_random_large(G):
    rng = np.random.default_rng(5)
    for (m, n) in [(1000, 777), (257, 4097), (33, 1)]:
        h = rnd(251, m, n, m + n)
        rows = tuple(sorted(rng.choice(m, size=m // 3, replace=False).tolist()))
        cols = tuple(sorted(rng.choice(n, size=max(n // 2, 1), replace=False).tolist()))
        s, r = G.rex(h, G.IndexSet(m, rows))
        ws, wr = R.rex(h, R.IndexSet(m, rows))
        assert s == ws and r == wr
        s, r = G.cex(h, G.IndexSet(n, cols))
        ws, wr = R.cex(h, R.IndexSet(n, cols))
        assert s == ws and r == wr
        u = tuple(int(x) for x in rng.integers(0, 2, m))
        b = rnd(251, u.count(0), n, 1)
        c = rnd(251, u.count(1), n, 2)
        assert G.rrf(u, b, c) == R.rrf(u, b, c)


def test_index_jobs_pinned(G, pinned):
    for c in pinned["unh"]:
        rho, u = G.unh(G.IndexSet(*c["rho1"][:1], tuple(c["rho1"][1])), G.IndexSet(c["rho2"][0], tuple(c["rho2"][1])))
        assert list(rho.members) == c["rho"] and list(u) == c["u"]
    for c in pinned["mkr"]:
        assert list(G.mkr(G.IndexSet(c["rho1"][0], tuple(c["rho1"][1])),
                          G.IndexSet(c["rho2"][0], tuple(c["rho2"][1])))) == c["u"]
    rho, u = G.un0(G.IndexSet(3, (0, 2)))
    assert rho == G.IndexSet(3, (0, 2)) and list(u) == [1, 1]


@pytest.mark.parametrize("zeros", [0, 1, 7, 300])
def test_crz_long_runs(G, zeros):
    """Column riffles whose map is long contiguous runs (the 16-byte run fast
    path of the gather, at every source alignment) against the restatement,
    including the pass-through when nothing is inserted."""
    rng = np.random.default_rng(zeros)
    m = rnd(251, 70, 3000, 9)
    lam = np.ones(3000 + zeros, np.uint8)
    lam[rng.choice(3000 + zeros, zeros, replace=False)] = 0
    lam = tuple(int(x) for x in lam)
    for view in (m, m[:, 5:]):   # the second: source rows not 16B-aligned at column 0
        view = np.ascontiguousarray(view)
        k = view.shape[1]
        lam2 = lam[: k + zeros]
        if sum(lam2) != k:
            lam2 = tuple([1] * k + [0] * zeros)
        got = G.crz(view, lam2, len(lam2))
        np.testing.assert_array_equal(got.numpy(), R.crz(view, lam2, len(lam2)))


def test_dma_selects_few_runs(G):
    """Large selects whose map is a few runs go to the copy engines
    (cudaMemcpy2DAsync / cudaMemset2DAsync): riffle inserting rows, a row
    split with rows missing, a widening by a zero part, two-operand column
    riffles -- all against the restatement."""
    rng = np.random.default_rng(3)
    b = rnd(7, 2300, 4000, 1)     # >= 8 MB outputs take the DMA path
    c = rnd(7, 2, 4000, 2)
    u = [0] * 2302
    u[5] = u[1900] = 1
    np.testing.assert_array_equal(G.rrf(tuple(u), b, c).numpy(), R.rrf(tuple(u), b, c))
    rho = G.IndexSet(2300, tuple(x for x in range(2300) if x not in (17, 2299)))
    sel, rest = G.rex(b, rho)
    want_sel, want_rest = R.rex(b, R.IndexSet(2300, [x for x in range(2300) if x not in (17, 2299)]))
    np.testing.assert_array_equal(sel.numpy(), want_sel)
    np.testing.assert_array_equal(rest.numpy(), want_rest)
    lam = tuple([1] * 1500 + [0] * 700 + [1] * 2500)
    np.testing.assert_array_equal(G.crz(b, lam, len(lam)).numpy(), R.crz(b, lam, len(lam)))
    gam = G.IndexSet(4000, tuple(range(0, 3000)))
    s2, r2 = G.cex(b, gam)
    np.testing.assert_array_equal(s2.numpy(), b[:, :3000])
    np.testing.assert_array_equal(r2.numpy(), b[:, 3000:])


# ------------------------------------------------------------------ K2 + recursion (ech)
@pytest.fixture(params=[0, 1], ids=["panel", "recursive"])
def mode(G, request):
    G.set_ech_mode(request.param)
    yield request.param
    G.set_ech_mode(0)


def check_ech(G, p, H, e, thr=None):
    o = oracle.oracle_rref(p, H)
    assert e.rank() == o["rank"]
    assert list(e.rho.members) == o["rho"].tolist()
    assert list(e.gamma.members) == o["gamma"].tolist()
    for key in "MKR":
        got = getattr(e, key)
        assert got.shape == o[key].shape, (key, got.shape, o[key].shape)
        np.testing.assert_array_equal(got.numpy(), o[key])


def test_ech_pinned(G, mode, pinned):
    f = G.FieldSpec(3)
    for c in pinned["ech"]:
        h = arr(c["h"])
        e = G.ech(f, h)
        r = len(c["gamma"])
        assert list(e.rho.members) == c["rho"] and list(e.gamma.members) == c["gamma"]
        assert e.M == arr(c["M"]).reshape(r, r)
        assert e.K == arr(c["K"]).reshape(h.shape[0] - r, r)
        assert e.R == arr(c["R"]).reshape(r, h.shape[1] - r)


def test_ech_empty_and_zero(G, mode):
    f = G.FieldSpec(3)
    for shape in [(0, 3), (3, 0), (0, 0)]:
        e = G.ech(f, np.zeros(shape, np.uint8))
        assert e.rank() == 0 and e.R.shape == (0, shape[1]) and e.K.shape == (shape[0], 0)
    e = G.ech(f, np.zeros((3, 4), np.uint8))
    assert e.rank() == 0 and e.K.shape == (3, 0) and e.R.shape == (0, 4)


@pytest.mark.parametrize("p", PRIMES)
def test_ech_random_shapes_and_thresholds(G, mode, p):
    f = G.FieldSpec(p)
    cases = [(1, 1), (4, 4), (5, 3), (3, 5), (16, 16), (33, 17), (100, 100), (200, 130), (130, 300)]
    for t, (m, n) in enumerate(cases):
        H = rnd(p, m, n, 100 + p + t)
        for thr in (1, 7, 64, 256):
            if thr == 1 and m * n > 2000:
                continue
            check_ech(G, p, H, G.ech(f, H, thr))
    low = oracle.random_product_matrix(p, 150, 140, 37, 7)
    check_ech(G, p, low, G.ech(f, low, 32))


@pytest.mark.parametrize("p", [3, 7, 251])
def test_ech_panel_window_fallbacks(G, p):
    """Panel shapes that defeat the general-p 64-row window (pivots more than
    64 rows below the first open row, free columns, pivotal rows inside the
    window) must give the same result as the full CTA algorithm."""
    G.set_ech_mode(0)
    f = G.FieldSpec(p)
    rng = np.random.default_rng(p)
    H = rnd(p, 300, 200, 1)
    H[:100] = 0                       # window of panel 0 sees zero rows only
    check_ech(G, p, H, G.ech(f, H))
    H = rnd(p, 300, 200, 2)
    H[:100, :64] = 0                  # panels 0-1 fall back, later panels use the window
    check_ech(G, p, H, G.ech(f, H))
    H = rnd(p, 90, 200, 3)
    H[:, rng.choice(200, 50, replace=False)] = 0   # free columns
    check_ech(G, p, H, G.ech(f, H))
    H = rnd(p, 400, 120, 4)
    H[rng.choice(400, 300, replace=False)] = 0     # sparse rows: windows skip zeros
    check_ech(G, p, H, G.ech(f, H))
    H = rnd(p, 2000, 96, 5)
    H[::3] = 0
    check_ech(G, p, H, G.ech(f, H))
    low = oracle.random_product_matrix(p, 500, 300, 70, 6)   # rank 70 < 300 columns
    check_ech(G, p, low, G.ech(f, low))


@pytest.mark.parametrize("p", [2, 3, 251])
@pytest.mark.parametrize("outer", [32, 96, 256])
def test_ech_two_level_outer_panels(G, p, outer):
    """The two-level device ECH (outer panels eliminated in a scratch with
    the row operator tracked in Y, one deep-K trailing contraction per outer
    panel) against the oracle on ragged, rank-deficient, zero-column and
    sparse-row blocks; outputs must not depend on the outer width."""
    G.set_ech_mode(0)
    f = G.FieldSpec(p)
    rng = np.random.default_rng(outer + p)
    G.set_ech_outer(outer)
    try:
        for t, (m, n) in enumerate([(300, 500), (520, 300), (257, 263), (64, 700), (1100, 300)]):
            H = rnd(p, m, n, 40 + t)
            check_ech(G, p, H, G.ech(f, H))
        H = rnd(p, 400, 330, 50)
        H[:, rng.choice(330, 90, replace=False)] = 0     # free columns
        H[rng.choice(400, 150, replace=False)] = 0       # zero rows
        check_ech(G, p, H, G.ech(f, H))
        H = rnd(p, 400, 300, 51)
        H[:120, :100] = 0                               # windows fall back
        check_ech(G, p, H, G.ech(f, H))
        low = oracle.random_product_matrix(p, 450, 380, 150, 52)  # rank 150
        check_ech(G, p, low, G.ech(f, low))
    finally:
        G.set_ech_outer(-1)


def test_ech_reference_fixtures(G, mode, ref_runs):
    for c in ref_runs["ech"]:
        H = np.array(c["H"], np.uint8).reshape(c["m"], c["n"])
        e = G.ech(G.FieldSpec(c["p"]), H, c["threshold"])
        assert e.rank() == c["rank"] and list(e.gamma.members) == c["gamma"] and list(e.rho.members) == c["rho"]
        for key in "MKR":
            np.testing.assert_array_equal(getattr(e, key).numpy(),
                                          np.array(c[key], np.uint8).reshape(getattr(e, key).shape))


@pytest.mark.parametrize("base", [8, 32, 128])
def test_ech_base_size_does_not_change_results(G, base):
    G.set_ech_base(base)
    try:
        H = rnd(5, 300, 260, 11)
        check_ech(G, 5, H, G.ech(G.FieldSpec(5), H))
    finally:
        G.set_ech_base(64)


def test_ech_large_block(G, mode):
    p = 2
    H = rnd(p, 1024, 1024, 3)
    e = G.ech(G.FieldSpec(p), H)
    check_ech(G, p, H, e)


# ------------------------------------------------------------------ K6
def test_generator_matches_reference(G, ref_runs):
    for g in ref_runs["generators"]:
        f = G.FieldSpec(g["p"])
        if g["kind"] == "random":
            got = G.random_matrix(f, g["m"], g["n"], g["seed"])
        else:
            got = G.random_product_matrix(f, g["m"], g["n"], g["inner"], g["seed"])
        np.testing.assert_array_equal(got.numpy(), np.array(g["C"], np.uint8).reshape(g["m"], g["n"]))
    for p, m, n, seed in [(3, 2000, 2000, 1), (251, 777, 1025, 9), (2, 64, 8192, 5)]:
        np.testing.assert_array_equal(G.random_matrix(G.FieldSpec(p), m, n, seed).numpy(),
                                      oracle.random_matrix(p, m, n, seed))
    np.testing.assert_array_equal(G.random_product_matrix(G.FieldSpec(7), 300, 280, 100, 4).numpy(),
                                  oracle.random_product_matrix(7, 300, 280, 100, 4))


@pytest.mark.parametrize("case", ["square2048", "tall1536", "wide1000x7500", "low2048", "zero_rows"])
def test_ech_gf2_split_vs_reference(G, case):
    """GF(2) blocks beyond the whole-block cluster kernel (> 1024 rows, or a
    packed [W | T] row beyond its nibble tables): the two-level path with one
    cluster launch per outer panel (mode 4), the same path with single-CTA
    panel steps (mode 2) and the reference's split rule (src/jobs.cpp:202-225)
    down to the cluster kernel (mode 0, the default), each bit-exact against
    the reference's own ech."""
    p = 2
    f = G.FieldSpec(p)
    rng = np.random.default_rng(7)
    if case == "square2048":
        H = rnd(p, 2048, 2048, 61)
    elif case == "tall1536":
        H = rnd(p, 1536, 900, 62)
    elif case == "wide1000x7500":
        H = rnd(p, 1000, 7500, 63)
    elif case == "low2048":
        P = rng.integers(0, 2, (2048, 1500)).astype(np.float64)
        Q = rng.integers(0, 2, (1500, 2048)).astype(np.float64)
        H = (P @ Q).astype(np.int64).__mod__(2).astype(np.uint8)
    else:
        H = rnd(p, 2100, 1100, 64)
        H[:700] = 0
        H[1500:1800] = H[100:400] ^ H[900:1200]
    want = oracle.ref_ech(p, H)
    outs = []
    try:
        for mode in (4, 2, 0):  # outer-panel cluster, single-CTA panel steps, split
            G.set_ech_mode(mode)
            outs.append(G.ech(f, H))
    finally:
        G.set_ech_mode(0)
    for e in outs:
        assert e.rank() == want["rank"]
        assert list(e.rho.members) == list(want["rho"]) and list(e.gamma.members) == list(want["gamma"])
        for key in "MKR":
            np.testing.assert_array_equal(getattr(e, key).numpy(), want[key])


@pytest.mark.parametrize("p", [2, 3, 251])
def test_ech_thin_blocks(G, mode, p):
    """Thin blocks (min(rows, cols) <= 32, the Chief's one-column / one-row
    ClearDowns) go to the one-launch base case: tall-thin and short-wide,
    random, sparse (mostly zero) and all-zero."""
    f = G.FieldSpec(p)
    for t, (m, n) in enumerate([(5000, 1), (3000, 4), (2000, 32), (1, 5000), (4, 3000), (32, 2000),
                                (8192, 1), (1, 8192)]):
        H = rnd(p, m, n, 500 + t)
        check_ech(G, p, H, G.ech(f, H))
        S = H.copy()
        S[np.random.default_rng(t).random(S.shape) < 0.995] = 0
        check_ech(G, p, S, G.ech(f, S))
        Z = np.zeros((m, n), np.uint8)
        Z[m // 2, n // 2] = 1
        check_ech(G, p, Z, G.ech(f, Z))
        check_ech(G, p, np.zeros((m, n), np.uint8), G.ech(f, np.zeros((m, n), np.uint8)))
