"""Pin the CPU oracle (C restatement + numpy task restatement) before trusting it.

Checks every oracle function against (1) the reference test suite's pinned
values (tests/golden/pinned.json) and (2) outputs of the reference library
itself (tests/golden/ref_runs.json, generated from oracle/_ref), and -- when
oracle/_ref is present -- against the live reference on more seeded cases.
CPU only.
"""
import numpy as np
import pytest

import oracle
from oracle import restate as R
from gfq_testutil import arr


def iset(x):
    return R.IndexSet(x[0], tuple(x[1]))


# ------------------------------------------------------------ generators / mad
def test_generators_match_reference_fixtures(ref_runs):
    for g in ref_runs["generators"]:
        if g["kind"] == "random":
            got = oracle.random_matrix(g["p"], g["m"], g["n"], g["seed"])
        else:
            got = oracle.random_product_matrix(g["p"], g["m"], g["n"], g["inner"], g["seed"])
        np.testing.assert_array_equal(got, np.array(g["C"], np.uint8).reshape(g["m"], g["n"]))


def test_splitmix_counter_form():
    # draw t of a stream is mix(seed + (t+1)*golden): the counter form the
    # device generator uses.
    import ctypes
    st = ctypes.c_uint64(12345)
    seq = [oracle.lib.gfo_splitmix_next(ctypes.byref(st)) for _ in range(5)]
    oracle.lib.gfo_splitmix_next.restype = ctypes.c_uint64
    st = ctypes.c_uint64(12345)
    seq = [oracle.lib.gfo_splitmix_next(ctypes.byref(st)) for _ in range(5)]
    for t in range(5):
        s2 = ctypes.c_uint64((12345 + t * 0x9E3779B97F4A7C15) & (2**64 - 1))
        assert oracle.lib.gfo_splitmix_next(ctypes.byref(s2)) == seq[t]


def test_mad_pinned(pinned):
    p = pinned["p"]
    for c in pinned["mul"]:
        np.testing.assert_array_equal(oracle.mad(p, arr(c["b"]), arr(c["c"])), arr(c["out"]))
    for c in pinned["mad"]:
        np.testing.assert_array_equal(oracle.mad(p, arr(c["b"]), arr(c["c"]), arr(c["a"])), arr(c["out"]))


@pytest.mark.parametrize("p", [2, 3, 7, 193, 251])
def test_mad_vs_numpy_int64(p):
    rng = np.random.default_rng(p)
    for (m, k, n) in [(7, 5, 9), (1, 1, 1), (3, 0, 4), (0, 3, 4), (16, 33, 8), (5, 300, 2)]:
        a = rng.integers(0, p, (m, k), dtype=np.int64)
        b = rng.integers(0, p, (k, n), dtype=np.int64)
        c = rng.integers(0, p, (m, n), dtype=np.int64)
        want = (c + a @ b) % p
        got = oracle.mad(p, a.astype(np.uint8), b.astype(np.uint8), c.astype(np.uint8))
        np.testing.assert_array_equal(got, want.astype(np.uint8))


def test_mad_shape_errors():
    with pytest.raises(ValueError):
        oracle.mad(3, np.zeros((2, 3), np.uint8), np.zeros((2, 3), np.uint8))
    with pytest.raises(ValueError):
        oracle.mad(3, np.zeros((2, 3), np.uint8), np.zeros((3, 3), np.uint8), np.zeros((2, 2), np.uint8))


# ------------------------------------------------------------ ech / oracle_rref
def test_ech_pinned(pinned):
    for c in pinned["ech"]:
        h = arr(c["h"])
        e = R.ech(3, h)
        r = len(c["gamma"])
        assert list(e.rho.members) == c["rho"] and list(e.gamma.members) == c["gamma"]
        np.testing.assert_array_equal(e.M, arr(c["M"]).reshape(r, r))
        np.testing.assert_array_equal(e.K, arr(c["K"]).reshape(h.shape[0] - r, r))
        np.testing.assert_array_equal(e.R, arr(c["R"]).reshape(r, h.shape[1] - r))


def test_ech_matches_reference_fixture_across_thresholds(ref_runs):
    # canonical ECH: the reference's recursive ech at any threshold equals the
    # sequential oracle on all five outputs
    for c in ref_runs["ech"]:
        H = np.array(c["H"], np.uint8).reshape(c["m"], c["n"])
        o = oracle.oracle_rref(c["p"], H)
        assert o["rank"] == c["rank"]
        assert o["rho"].tolist() == c["rho"] and o["gamma"].tolist() == c["gamma"]
        for key in "MKR":
            np.testing.assert_array_equal(o[key], np.array(c[key], np.uint8).reshape(o[key].shape))


def test_ech_empty_shapes():
    for shape in [(0, 3), (3, 0), (0, 0)]:
        e = R.ech(3, np.zeros(shape, np.uint8))
        assert e.rank() == 0
        assert e.R.shape == (0, shape[1]) and e.K.shape == (shape[0], 0)


def check_identity(p, h, e):
    """reference tests/test_jobs.cpp:35-70 (`check_ech_identity`)."""
    r = e.rank()
    sel, rest = R.rex(h, e.rho)
    perm = np.vstack([sel, rest])
    cs, cr = R.cex(perm, e.gamma)
    permuted = np.hstack([cs, cr])
    top = R.mul(p, e.M, permuted[:r])
    bottom = R.mad(p, permuted[r:], e.K, permuted[:r])
    want = np.zeros((r, h.shape[1]), np.uint8)
    want[np.arange(r), np.arange(r)] = p - 1
    want[:, r:] = e.R
    np.testing.assert_array_equal(top, want)
    assert not bottom.any()


@pytest.mark.parametrize("p", [2, 3, 193, 251])
def test_ech_identity_random(p):
    for seed, (m, n) in enumerate([(1, 1), (4, 4), (5, 3), (3, 5), (16, 16), (33, 17)]):
        h = oracle.random_matrix(p, m, n, 100 + p + seed)
        check_identity(p, h, R.ech(p, h))
    low = oracle.random_product_matrix(p, 12, 12, 3, 7)
    check_identity(p, low, R.ech(p, low))


# ------------------------------------------------------------ small jobs
def test_index_jobs_pinned(pinned):
    for c in pinned["unh"]:
        rho, u = R.unh(iset(c["rho1"]), iset(c["rho2"]))
        assert list(rho.members) == c["rho"] and list(u) == c["u"]
    for c in pinned["mkr"]:
        assert list(R.mkr(iset(c["rho1"]), iset(c["rho2"]))) == c["u"]
    with pytest.raises(ValueError):
        R.unh(R.IndexSet(4, (0,)), R.IndexSet(4, (0,)))
    with pytest.raises(ValueError):
        R.mkr(R.IndexSet(4, (2,)), R.IndexSet(4, (0, 3)))


def test_riffles():
    # reference tests/test_jobs.cpp:248-318
    np.testing.assert_array_equal(R.rrf((0, 1, 0), arr([[1, 1], [2, 2]]), arr([[0, 0]])),
                                  arr([[1, 1], [0, 0], [2, 2]]))
    np.testing.assert_array_equal(R.crz(arr([[1], [2]]), (1, 0), 2), arr([[1, 0], [2, 0]]))
    np.testing.assert_array_equal(R.adi(np.zeros((2, 3), np.uint8), (1, 0, 1)), arr([[1, 0, 0], [0, 0, 1]]))
    with pytest.raises(ValueError):
        R.crz(arr([[1, 2, 0], [0, 1, 2]]), (1, 1), 2)
    with pytest.raises(ValueError):
        R.adi(np.zeros((1, 3), np.uint8), (1, 0, 1))
    h = oracle.random_matrix(7, 6, 4, 19)
    rho = R.IndexSet(6, (1, 3, 4))
    sel, rest = R.rex(h, rho)
    u = tuple(1 if t in rho.members else 0 for t in range(6))
    np.testing.assert_array_equal(R.rrf(u, rest, sel), h)


# ------------------------------------------------------------ tasks (paper 6x6)
def test_task_walkthrough_pinned(pinned):
    """reference tests/test_tasks.cpp:295-372 chain, every intermediate."""
    p = 3
    C00, C01, C10, C11 = (arr(pinned[k]) for k in ("C00", "C01", "C10", "C11"))
    W = pinned["walkthrough"]
    d0_v0, a00 = R.clear_down(p, C00, R.PkgD(), 0)
    cd0 = pinned["clear_down_0"]
    assert list(d0_v0.gamma.members) == cd0["gamma"]
    np.testing.assert_array_equal(d0_v0.R, arr(cd0["R"]))
    np.testing.assert_array_equal(a00.M, arr(cd0["M"]))
    np.testing.assert_array_equal(a00.K, arr(cd0["K"]))
    e0_v0 = R.extend(a00, None, 0)
    c01_v1, b01_v0 = R.update_row(p, a00, C01, None, 0)
    np.testing.assert_array_equal(b01_v0, arr(pinned["update_row_0"]["B"]))
    np.testing.assert_array_equal(c01_v1, arr(pinned["update_row_0"]["C"]))
    k00, m00 = R.update_row_trafo(p, a00, None, None, e0_v0, 0, 0, 0)
    d1_v0, a01 = R.clear_down(p, c01_v1, R.PkgD(), 0)
    e0_v1 = R.extend(a01, e0_v0, 1)
    k00, m = R.update_row_trafo(p, a01, k00, None, e0_v1, 0, 0, 1)
    np.testing.assert_array_equal(m, arr(W["m01_first"]))
    assert list(d1_v0.gamma.members) == W["d1_v0"]["gamma"]
    np.testing.assert_array_equal(d1_v0.R, arr(W["d1_v0"]["R"]))
    d0_v1, a10 = R.clear_down(p, C10, d0_v0, 1)
    cd1 = pinned["clear_down_1"]
    np.testing.assert_array_equal(a10.A, arr(cd1["A"]))
    np.testing.assert_array_equal(a10.E, arr(cd1["E"]))
    assert list(a10.lam) == cd1["lambda"]
    e1_v0 = R.extend(a10, None, 0)
    c11_v1, b01_v1 = R.update_row(p, a10, C11, b01_v0, 1)
    np.testing.assert_array_equal(b01_v1, arr(pinned["update_row_1"]["B"]))
    np.testing.assert_array_equal(c11_v1, arr(pinned["update_row_1"]["C"]))
    k10, m00_v1 = R.update_row_trafo(p, a10, None, m00, e1_v0, 1, 0, 0)
    k11, m01 = R.update_row_trafo(p, a10, None, None, e1_v0, 1, 1, 0)
    np.testing.assert_array_equal(m00_v1, arr(W["m00_v1"]))
    np.testing.assert_array_equal(m01, arr(W["m01"]))
    d1_v1, a11 = R.clear_down(p, c11_v1, d1_v0, 1)
    e1_v1 = R.extend(a11, e1_v0, 1)
    k10_v2, m10_v1 = R.update_row_trafo(p, a11, k10, arr(W["m01_first"]), e0_v1, 1, 0, 1)
    k11_v2, m11 = R.update_row_trafo(p, a11, k11, None, e1_v1, 1, 1, 1)
    np.testing.assert_array_equal(m10_v1, arr(W["m10_v1"]))
    np.testing.assert_array_equal(k10_v2, arr(W["k10_v2"]))
    np.testing.assert_array_equal(m11, arr(W["m11"]))
    np.testing.assert_array_equal(k11_v2, arr(W["k11_v2"]))
    m00_len = R.row_lengthen(m00_v1, e0_v0, e0_v1)
    m01_len = R.row_lengthen(m01, e1_v0, e1_v1)
    np.testing.assert_array_equal(m00_len, arr(W["m00_len"]))
    np.testing.assert_array_equal(m01_len, arr(W["m01_len"]))
    r11 = R.copy_d(d1_v1)
    x01, r01_v0 = R.pre_clear_up(b01_v1, d1_v1)
    np.testing.assert_array_equal(r11, arr(W["r11"]))
    np.testing.assert_array_equal(R.clear_up(p, r01_v0, x01, r11), arr(W["r01"]))
    np.testing.assert_array_equal(R.clear_up(p, m00_len, x01, m10_v1), arr(W["m00_f"]))
    np.testing.assert_array_equal(R.clear_up(p, m01_len, x01, m11), arr(W["m01_f"]))


def compare_outputs(got, want_run):
    """got: restate.Output; want_run: a ref_runs.json record."""
    assert got.rank == want_run["rank"]
    assert [list(s.members) for s in got.upsilon] == want_run["upsilon"]
    assert [list(s.members) for s in got.varrho] == want_run["varrho"]
    for key, v in want_run["R"].items():
        j, l = map(int, key.split(","))
        np.testing.assert_array_equal(got.R_blocks[(j, l)], arr(v))
    if want_run.get("with_transform", True):
        for key, v in want_run["TM"].items():
            j, h = map(int, key.split(","))
            np.testing.assert_array_equal(got.T_M_blocks[(j, h)], arr(v))
        for key, v in want_run["TK"].items():
            i, h = map(int, key.split(","))
            np.testing.assert_array_equal(got.T_K_blocks[(i, h)], arr(v))
        np.testing.assert_array_equal(got.materialize_transform(), np.array(want_run["T"], np.uint8))


def test_paper_example_full_output(pinned):
    C6 = arr(pinned["C6"])
    want = pinned["C6_out"]
    for out in (R.echelonize(3, C6, 3), R.blocked_from_oracle(3, C6, 3)):
        assert out.rank == want["rank"]
        assert [list(s.members) for s in out.upsilon] == want["upsilon"]
        assert [list(s.members) for s in out.varrho] == want["varrho"]
        for k, v in want["R"].items():
            np.testing.assert_array_equal(out.R_blocks[tuple(map(int, k.split(",")))], arr(v))
        for k, v in want["TM"].items():
            np.testing.assert_array_equal(out.T_M_blocks[tuple(map(int, k.split(",")))], arr(v))
        for k, v in want["TK"].items():
            np.testing.assert_array_equal(out.T_K_blocks[tuple(map(int, k.split(",")))], arr(v))
        np.testing.assert_array_equal(out.assembled_R(), arr(want["assembled_R"]))
        np.testing.assert_array_equal(out.materialize_transform(), arr(want["T"]))


def test_restated_chief_matches_reference_runs(ref_runs):
    for run in ref_runs["echelonize"]:
        C = np.array(run["C"], np.uint8).reshape(run["m"], run["n"])
        got = R.echelonize(run["p"], C, run["block"], run["with_transform"])
        compare_outputs(got, run)
        if run["with_transform"]:
            compare_outputs(R.blocked_from_oracle(run["p"], C, run["block"]), run)


def test_identity_and_zero_inputs():
    # reference tests/test_chief.cpp:196-236
    idm = np.eye(6, dtype=np.uint8)
    out = R.echelonize(3, idm, 2)
    assert out.rank == 6
    np.testing.assert_array_equal(out.materialize_transform(), 2 * np.eye(6, dtype=np.uint8))
    z = np.zeros((4, 5), np.uint8)
    out = R.echelonize(5, z, 2)
    assert out.rank == 0
    np.testing.assert_array_equal(out.materialize_transform(), np.eye(4, dtype=np.uint8))


@pytest.mark.skipif(oracle.ref is None, reason="oracle/_ref not built")
def test_restatement_vs_live_reference_more_cases():
    rng = np.random.default_rng(1)
    for t in range(12):
        p = int(rng.choice([2, 3, 5, 7, 251]))
        m, n = int(rng.integers(1, 30)), int(rng.integers(1, 30))
        blk = int(rng.integers(1, 12))
        if t % 3 == 0:
            C = oracle.ref_random_product_matrix(p, m, n, int(rng.integers(0, min(m, n) + 1)), 100 + t)
        else:
            C = oracle.ref_random_matrix(p, m, n, 100 + t)
        ref = oracle.ref_echelonize(p, C, blk)
        got = R.blocked_from_oracle(p, C, blk)
        assert got.rank == ref.rank
        for j in range(ref.b):
            assert list(got.upsilon[j].members) == ref.upsilon(j).tolist()
            for l in range(j, ref.b):
                np.testing.assert_array_equal(got.R_blocks[(j, l)], ref.block(0, j, l))
        np.testing.assert_array_equal(got.materialize_transform(), ref.materialize_transform())


@pytest.mark.skipif(oracle.ref is None, reason="oracle/_ref not built")
@pytest.mark.parametrize("p", [2, 3, 251])
def test_reference_tk_support_is_lex_first(p):
    """The structural pin used for cfg5s (tests/test_gpu_configs.py): in the
    reference's own output every T_K row (a non-selected row t) is supported
    only on selected rows of smaller index -- varrho is the
    lexicographically-first row basis (src/chief.cpp:436-460)."""
    rng = np.random.default_rng(p)
    for t, (m, n, r, block) in enumerate([(60, 50, 20, 16), (90, 40, 35, 32), (64, 64, 64, 16)]):
        P = oracle.random_matrix(p, m, r, 300 + t)
        Q = oracle.random_matrix(p, r, n, 400 + t)
        C = oracle.mad(p, P, Q)
        C[rng.choice(m, m // 5, replace=False)] = 0
        ref = oracle.ref_echelonize(p, C, block, threads=2)
        for i in range(ref.a):
            sel = ref.varrho(i).astype(np.int64)
            rows_i = min(block, m - i * block)
            non = np.setdiff1d(np.arange(rows_i), sel)
            tk = ref.block(2, i, i)
            assert tk.shape == (len(non), len(sel))
            if tk.size:
                assert not np.any(tk[sel[None, :] > non[:, None]])
