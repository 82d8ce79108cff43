"""GPU parity of the full echelonize path (ChopMatrix -> Steps 1-3 on the
CUDA stream DAG -> EchelonOutput) against the reference and the oracle.

Bit-exact on rank, pivot columns (upsilon), selected rows (varrho), every R /
T_M / T_K block and the materialised transformation; plus the
size-independent defining identity T.C = [[-1, R], [0, 0]] at sizes where
the scalar oracle is too slow.
"""
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


def compare(out, want, with_transform=True):
    """out: gfrref.EchelonOutput (device); want: restate.Output or ref fixture dict."""
    if isinstance(want, dict):
        assert out.rank == want["rank"]
        assert [list(s.members) for s in out.upsilon] == want["upsilon"]
        assert [list(s.members) for s in out.varrho] == want["varrho"]
        for key, v in want["R"].items():
            j, l = map(int, key.split(","))
            np.testing.assert_array_equal(out.block(0, j, l).numpy(), arr(v))
        np.testing.assert_array_equal(out.assembled_R().numpy(),
                                      np.array(want["assembled_R"], np.uint8).reshape(out.rank,
                                                                                      want["n"] - out.rank))
        if with_transform:
            for key, v in want["TM"].items():
                j, h = map(int, key.split(","))
                np.testing.assert_array_equal(out.block(1, j, h).numpy(), arr(v))
            for key, v in want["TK"].items():
                i, h = map(int, key.split(","))
                np.testing.assert_array_equal(out.block(2, i, h).numpy(), arr(v))
            np.testing.assert_array_equal(out.materialize_transform().numpy(), np.array(want["T"], np.uint8))
        return
    assert out.rank == want.rank
    assert [s.members for s in out.upsilon] == [s.members for s in want.upsilon]
    assert [s.members for s in out.varrho] == [s.members for s in want.varrho]
    b, a = len(want.col_parts), len(want.row_parts)
    for j in range(b):
        for l in range(j, b):
            np.testing.assert_array_equal(out.block(0, j, l).numpy(), want.R_blocks[(j, l)])
    if with_transform:
        for j in range(b):
            for h in range(a):
                np.testing.assert_array_equal(out.block(1, j, h).numpy(), want.T_M_blocks[(j, h)])
        for i in range(a):
            for h in range(i + 1):
                np.testing.assert_array_equal(out.block(2, i, h).numpy(), want.T_K_blocks[(i, h)])
        np.testing.assert_array_equal(out.materialize_transform().numpy(), want.materialize_transform())


def test_paper_example(G, pinned):
    C6 = arr(pinned["C6"])
    want = pinned["C6_out"]
    for threads in (1, 3):
        out = G.echelonize(C6, G.FieldSpec(3), G.EchelonizeOptions(block=3, threads=threads, collect_trace=True,
                                                                   fuse=False))
        assert out.rank == want["rank"]
        assert [list(s.members) for s in out.upsilon] == want["upsilon"]
        assert [list(s.members) for s in out.varrho] == want["varrho"]
        for k, v in want["R"].items():
            assert out.block(0, *map(int, k.split(","))) == arr(v)
        for k, v in want["TM"].items():
            assert out.block(1, *map(int, k.split(","))) == arr(v)
        for k, v in want["TK"].items():
            assert out.block(2, *map(int, k.split(","))) == arr(v)
        assert out.assembled_R() == arr(want["assembled_R"])
        assert out.materialize_transform() == arr(want["T"])
        assert out.global_upsilon() == [0, 1, 2, 3, 5] and out.global_varrho() == [0, 1, 2, 3, 5]
        tr = out.trace()
        counts = {}
        for t in tr:
            counts[t["kind"]] = counts.get(t["kind"], 0) + 1
        assert len(tr) == want["task_counts"]["total"]
        for k, v in want["task_counts"].items():
            if k != "total":
                assert counts.get(k, 0) == v, k
        # ClearDown details = new pivots per block column (test_chief.cpp:436-454)
        per_col = {}
        for t in tr:
            if t["kind"] == "ClearDown":
                per_col[t["j"]] = per_col.get(t["j"], 0) + t["detail"]
        assert per_col == {0: 3, 1: 2}
    lean = G.echelonize(C6, G.FieldSpec(3), G.EchelonizeOptions(block=3, with_transform=False, collect_trace=True,
                                                                 fuse=False))
    assert len(lean.trace()) == want["task_counts_no_transform"]["total"]
    assert lean.rank == 5 and lean.assembled_R() == arr(want["assembled_R"])


def test_reference_run_fixtures(G, ref_runs):
    for run in ref_runs["echelonize"]:
        C = np.array(run["C"], np.uint8).reshape(run["m"], run["n"])
        for threads in (1, 4):
            out = G.echelonize(C, G.FieldSpec(run["p"]),
                               G.EchelonizeOptions(block=run["block"], threads=threads,
                                                   with_transform=run["with_transform"]))
            compare(out, run, run["with_transform"])


def test_identity_zero_and_empty(G):
    idm = np.eye(6, dtype=np.uint8)
    out = G.echelonize(idm, G.FieldSpec(3), G.EchelonizeOptions(block=2))
    assert out.rank == 6
    np.testing.assert_array_equal(out.materialize_transform().numpy(), 2 * np.eye(6, dtype=np.uint8))
    z = np.zeros((4, 5), np.uint8)
    out = G.echelonize(z, G.FieldSpec(5), G.EchelonizeOptions(block=2))
    assert out.rank == 0
    np.testing.assert_array_equal(out.materialize_transform().numpy(), np.eye(4, dtype=np.uint8))
    for shape in [(0, 5), (5, 0), (0, 0)]:
        out = G.echelonize(np.zeros(shape, np.uint8), G.FieldSpec(3), G.EchelonizeOptions(block=2))
        assert out.rank == 0


@pytest.mark.parametrize("p,m,n,block,kind", [
    (2, 300, 300, 64, "random"), (3, 257, 301, 48, "random"), (7, 320, 256, 80, "product"),
    (251, 200, 200, 50, "random"), (5, 190, 230, 37, "product"), (2, 256, 256, 256, "random"),
])
def test_random_vs_oracle(G, p, m, n, block, kind):
    C = oracle.random_matrix(p, m, n, m + n) if kind == "random" else \
        oracle.random_product_matrix(p, m, n, min(m, n) // 3, m + n)
    out = G.echelonize(C, G.FieldSpec(p), G.EchelonizeOptions(block=block, threads=4))
    compare(out, R.blocked_from_oracle(p, C, block))


def test_block_size_and_thread_independence(G):
    p = 5
    C = oracle.random_matrix(p, 120, 120, 0xB10C)
    base = G.echelonize(C, G.FieldSpec(p), G.EchelonizeOptions(block=120))
    T0 = base.materialize_transform().numpy()
    for block, threads in [(1, 1), (7, 2), (13, 4), (40, 8)]:
        out = G.echelonize(C, G.FieldSpec(p), G.EchelonizeOptions(block=block, threads=threads))
        assert out.rank == base.rank and out.global_upsilon() == base.global_upsilon()
        assert out.assembled_R() == base.assembled_R()
        np.testing.assert_array_equal(out.materialize_transform().numpy(), T0)


def _identity_check(G, p, C, out):
    """T.C == [[-1, R], [0, 0]] (reference src/chief.cpp:566-588), with T and
    C on the device and the product on K1."""
    f = G.FieldSpec(p)
    T = out.materialize_transform()
    P = G.mul(f, T, C).numpy()
    r = out.rank
    ups = out.global_upsilon()
    rest = [c for c in range(C.cols if isinstance(C, G.Matrix) else C.shape[1]) if c not in set(ups)]
    Rm = out.assembled_R().numpy()
    want = np.zeros_like(P)
    want[np.arange(r), ups] = p - 1
    if rest:
        want[:r][:, rest] = Rm
    np.testing.assert_array_equal(P, want)


@pytest.mark.skipif(oracle.ref is None, reason="oracle/_ref not built")
def test_cfg1_vs_reference_library(G):
    """configs[0]: GF(3) 2000x2000, block 500 -- bit-exact against the
    reference's own blocked echelonize (oracle/_ref)."""
    p, m, block = 3, 2000, 500
    C = oracle.random_matrix(p, m, m, 1)
    ref = oracle.ref_echelonize(p, C, block, threads=8)
    Cd = G.random_matrix(G.FieldSpec(p), m, m, 1)
    out = G.echelonize(Cd, G.FieldSpec(p), G.EchelonizeOptions(block=block, threads=4))
    assert out.rank == ref.rank == 1999
    for j in range(ref.b):
        assert list(out.upsilon[j].members) == ref.upsilon(j).tolist()
        for l in range(j, ref.b):
            np.testing.assert_array_equal(out.block(0, j, l).numpy(), ref.block(0, j, l))
        for h in range(ref.a):
            np.testing.assert_array_equal(out.block(1, j, h).numpy(), ref.block(1, j, h))
    for i in range(ref.a):
        assert list(out.varrho[i].members) == ref.varrho(i).tolist()
        for h in range(i + 1):
            np.testing.assert_array_equal(out.block(2, i, h).numpy(), ref.block(2, i, h))
    np.testing.assert_array_equal(out.materialize_transform().numpy(), ref.materialize_transform())


@pytest.mark.parametrize("p,m,n,block", [(2, 2048, 2048, 256), (251, 1536, 1024, 512), (7, 1024, 1536, 256)])
def test_defining_identity_medium(G, p, m, n, block):
    C = G.random_matrix(G.FieldSpec(p), m, n, 77)
    out = G.echelonize(C, G.FieldSpec(p), G.EchelonizeOptions(block=block, threads=4))
    assert out.rank == min(m, n) or p == 2
    _identity_check(G, p, C, out)


def test_dependency_race_regression(G):
    """A rank-deficient input whose ClearDowns often have no new pivots (no
    device work of their own): their packages must still be ordered after
    their inputs.  Slow SIMT contractions and 8 workers widen the window;
    every repetition must give the same output (a lost wait showed up as
    spurious pivots in ~20% of runs)."""
    import hashlib
    p, half, n, block = 2, 512, 1024, 128
    f = G.FieldSpec(p)
    top = G.random_matrix(f, half, n, 5).numpy()
    top[:, :block] = 0
    comb = G.random_matrix(f, half, half, 6)
    bottom = G.mul(f, comb, G.Matrix.from_numpy(top)).numpy()
    C = G.Matrix.from_numpy(np.vstack([top, bottom]))
    want = None
    G.set_mad_policy(1)
    try:
        for _ in range(12):
            out = G.echelonize(C, f, G.EchelonizeOptions(block=block, threads=8))
            buf = np.zeros(out.block_bytes(), np.uint8)
            out.download_blocks(buf)
            got = (out.rank, hashlib.sha1(buf.tobytes()).hexdigest())
            want = want or got
            assert got == want
    finally:
        G.set_mad_policy(0)
    assert want[0] <= half


@pytest.mark.parametrize("p,m,n,block,kind,wt", [
    (2, 300, 300, 64, "random", True), (3, 257, 301, 48, "random", True), (7, 320, 256, 80, "product", True),
    (251, 200, 230, 50, "random", True), (5, 190, 230, 37, "product", True), (2, 512, 384, 64, "product", False),
    (3, 96, 400, 32, "random", True), (2, 64, 64, 64, "random", True),
])
def test_fused_plan_matches_reference_grid(G, p, m, n, block, kind, wt):
    """The fused single-GPU plan (wide UpdateRow / ClearUp jobs on panels)
    computes exactly the reference task grid's values."""
    f = G.FieldSpec(p)
    C = G.random_matrix(f, m, n, 21) if kind == "random" else G.random_product_matrix(f, m, n, min(m, n) // 3, 21)
    ref = G.echelonize(C, f, G.EchelonizeOptions(block=block, threads=3, with_transform=wt, fuse=False))
    fus = G.echelonize(C, f, G.EchelonizeOptions(block=block, threads=3, with_transform=wt, fuse=True))
    assert fus.rank == ref.rank
    assert [s.members for s in fus.upsilon] == [s.members for s in ref.upsilon]
    assert [s.members for s in fus.varrho] == [s.members for s in ref.varrho]
    a, b = len(ref.chop.row_parts), len(ref.chop.col_parts)
    for j in range(b):
        for l in range(j, b):
            np.testing.assert_array_equal(fus.block(0, j, l).numpy(), ref.block(0, j, l).numpy())
        if wt:
            for h in range(a):
                np.testing.assert_array_equal(fus.block(1, j, h).numpy(), ref.block(1, j, h).numpy())
    if wt:
        for i in range(a):
            for h in range(i + 1):
                np.testing.assert_array_equal(fus.block(2, i, h).numpy(), ref.block(2, i, h).numpy())
    kinds = {t["kind"] for t in G.echelonize(C, f, G.EchelonizeOptions(block=block, with_transform=wt,
                                                                       collect_trace=True)).trace()}
    if b > 2:
        assert "UpdateRowW" in kinds and "ClearUpRW" in kinds
    if wt and a > 1:
        assert "UpdateRowTrafoW" in kinds


@pytest.mark.parametrize("p,m,n,block,kind,wt,fuse", [
    (2, 300, 260, 64, "random", True, True), (7, 250, 310, 48, "product", True, True),
    (3, 200, 200, 50, "random", False, True), (251, 130, 170, 40, "random", True, False),
    (2, 96, 96, 96, "random", True, True)])
def test_early_download_matches_download_blocks(G, p, m, n, block, kind, wt, fuse):
    """echelonize(host C, host_out=buf) streams every final block into buf
    while Step 3 runs; the bytes equal gfq_output_download_blocks'."""
    C = oracle.random_matrix(p, m, n, 4) if kind == "random" else oracle.random_product_matrix(p, m, n, 30, 4)
    opts = G.EchelonizeOptions(block=block, threads=3, with_transform=wt, fuse=fuse)
    ref = G.echelonize(C, G.FieldSpec(p), opts)
    want = np.zeros(ref.block_bytes(), np.uint8)
    ref.download_blocks(want)
    buf = np.full(ref.block_bytes() + 7, 0xAB, np.uint8)
    out = G.echelonize(C, G.FieldSpec(p), opts, host_out=buf)
    assert out.rank == ref.rank
    np.testing.assert_array_equal(buf[: want.size], want)
    assert (buf[want.size:] == 0xAB).all()
    if want.size:
        with pytest.raises(Exception, match="too small"):
            G.echelonize(C, G.FieldSpec(p), opts, host_out=np.zeros(want.size - 1, np.uint8))


def test_concurrent_runs_share_the_executor_pools(G):
    """Several host threads echelonize at once: the process-wide worker-thread
    and stream pools (csrc/host/scheduler.cpp run_on_workers / acquire_stream)
    hand each run its own workers and streams; every result must equal the
    same run made alone, over several rounds (pooled streams are reused)."""
    import threading
    cases = [(3, 700, 650, 128), (2, 1500, 1400, 256), (7, 600, 900, 100), (251, 512, 512, 128)]
    inputs = [(p, oracle.random_matrix(p, m, n, 40 + q), block) for q, (p, m, n, block) in enumerate(cases)]
    alone = []
    for p, C, block in inputs:
        out = G.echelonize(C, G.FieldSpec(p), G.EchelonizeOptions(block=block, threads=3))
        alone.append((out.rank, out.assembled_R().numpy(), out.materialize_transform().numpy()))
    for _ in range(3):
        got, errs = [None] * len(inputs), []

        def body(q):
            try:
                p, C, block = inputs[q]
                out = G.echelonize(C, G.FieldSpec(p), G.EchelonizeOptions(block=block, threads=3))
                got[q] = (out.rank, out.assembled_R().numpy(), out.materialize_transform().numpy())
            except Exception as e:  # noqa: BLE001
                errs.append(e)

        th = [threading.Thread(target=body, args=(q,)) for q in range(len(inputs))]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout=300)
        assert not errs, errs
        for q in range(len(inputs)):
            assert got[q][0] == alone[q][0]
            np.testing.assert_array_equal(got[q][1], alone[q][1])
            np.testing.assert_array_equal(got[q][2], alone[q][2])


STEP1 = {"ClearDown", "UpdateRow", "UpdateRowTrafo", "Extend", "UpdateRowW", "UpdateRowTrafoW"}
STEP3 = {"Copy", "PreClearUp", "ClearUp", "ClearUpRW", "ClearUpMW"}


@pytest.mark.parametrize("threads,fuse", [(1, False), (1, True), (4, True)])
def test_memory_stability_acceptance_criterion6(G, threads, fuse):
    """The reference's acceptance criterion 6 (tests/acceptance.cpp:480-520)
    on the same input: 2048^2 GF(3), seed 0x6eed, block 256, with trace --
    peak live package bytes <= 4x the input, and the Step-3 peak <= 1.6x the
    Step-1 peak (the refcounted release keeps Step 3 from growing)."""
    p, n = 3, 2048
    C = G.random_matrix(G.FieldSpec(p), n, n, 0x6EED)
    out = G.echelonize(C, G.FieldSpec(p), G.EchelonizeOptions(block=256, threads=threads, collect_trace=True,
                                                              fuse=fuse))
    rep = out.report()
    input_bytes = n * n
    step1 = max((t["live_bytes"] for t in out.trace() if t["kind"] in STEP1), default=0)
    step3 = max((t["live_bytes"] for t in out.trace() if t["kind"] in STEP3), default=0)
    assert step1 > 0
    assert rep["peak_live_bytes"] <= 4.0 * input_bytes, (rep["peak_live_bytes"], input_bytes)
    assert step3 <= 1.6 * step1, (step3, step1)


@pytest.fixture
def host_pack(G):
    G.set_host_pack(True)
    yield
    G.set_host_pack(False)


@pytest.mark.parametrize("m,n,block", [(333, 517, 100), (1000, 70, 64), (64, 1000, 200), (517, 333, 517)])
def test_gf2_host_buffers_cross_pcie_packed(G, host_pack, m, n, block):
    """GF(2) host buffers travel packed 8:1 when asked (csrc/host/hostpack.cpp
    + kernels/bits.cu): the host-input run equals the device-input run, the
    streamed host_out equals gfq_output_download_blocks, and the PCIe byte
    counts are the packed sizes (rows padded to 8-byte words)."""
    f = G.FieldSpec(2)
    C = oracle.random_matrix(2, m, n, 11)
    opts = G.EchelonizeOptions(block=block, threads=3, with_transform=True)
    dev = G.echelonize(G.Matrix.from_numpy(C), f, opts)
    want = np.zeros(dev.block_bytes(), np.uint8)
    dev.download_blocks(want)
    buf = np.full(dev.block_bytes() + 5, 0xCD, np.uint8)
    out = G.echelonize(C, f, opts, host_out=buf)
    assert out.rank == dev.rank
    np.testing.assert_array_equal(buf[: want.size], want)
    assert (buf[want.size:] == 0xCD).all()
    h2d, d2h = G.last_transfer_bytes()
    assert h2d == m * ((n + 63) // 64 * 8)
    assert 0 < d2h <= want.size // 8 + 8 * 64 * 64 and d2h < want.size


@pytest.mark.parametrize("stride", [2, 3])
@pytest.mark.parametrize("m,n,block", [(333, 517, 100), (517, 333, 64)])
def test_gf2_host_buffers_hybrid_packing(G, stride, m, n, block):
    """Hybrid transfers (gfq_set_host_pack(N >= 2)): every N-th block row and
    output block packed, the rest as bytes -- same outputs, PCIe bytes between
    the all-packed and the all-bytes counts."""
    f = G.FieldSpec(2)
    C = oracle.random_matrix(2, m, n, 13)
    opts = G.EchelonizeOptions(block=block, threads=3, with_transform=True)
    dev = G.echelonize(G.Matrix.from_numpy(C), f, opts)
    want = np.zeros(dev.block_bytes(), np.uint8)
    dev.download_blocks(want)
    buf = np.full(dev.block_bytes() + 5, 0xCD, np.uint8)
    G.set_host_pack(stride)
    try:
        out = G.echelonize(C, f, opts, host_out=buf)
        h2d, d2h = G.last_transfer_bytes()
    finally:
        G.set_host_pack(False)
    assert out.rank == dev.rank
    np.testing.assert_array_equal(buf[: want.size], want)
    assert (buf[want.size:] == 0xCD).all()
    assert m * ((n + 63) // 64 * 8) < h2d < m * n
    assert d2h < want.size


@pytest.mark.parametrize("p,m,n,block,rank", [(2, 700, 650, 128, 300), (7, 520, 600, 96, 0), (2, 512, 512, 64, 0)])
def test_row_lengthen_in_two_halves(G, monkeypatch, p, m, n, block, rank):
    """GFQ_RL_SPLIT=1 (chief.cpp / scheduler.cpp RowLengthen c0 = -3 / -4: parts
    h < a-1 widened early into a full-stride panel, part a-1 appended in
    place) gives byte-identical outputs to the one-piece RowLengthen."""
    f = G.FieldSpec(p)
    rng = np.random.default_rng(5)
    if rank:
        C = (rng.integers(0, p, (m, rank)) @ rng.integers(0, p, (rank, n)) % p).astype(np.uint8)
    else:
        C = oracle.random_matrix(p, m, n, 21)
    opts = G.EchelonizeOptions(block=block, threads=3, with_transform=True)
    outs = []
    for split in ("0", "1"):
        monkeypatch.setenv("GFQ_RL_SPLIT", split)
        o = G.echelonize(G.Matrix.from_numpy(C), f, opts)
        buf = np.zeros(o.block_bytes(), np.uint8)
        o.download_blocks(buf)
        outs.append((o.rank, buf))
    assert outs[0][0] == outs[1][0]
    np.testing.assert_array_equal(outs[0][1], outs[1][1])


def test_host_buffers_cross_pcie_as_bytes_by_default(G):
    C = oracle.random_matrix(2, 200, 300, 12)
    G.echelonize(C, G.FieldSpec(2), G.EchelonizeOptions(block=64))
    assert G.last_transfer_bytes()[0] == 200 * 300
