"""GPU tests of the sharded Chief executor (csrc/host/dist.cpp) on one B200.

`world` loopback ranks run as threads of this process, each with its own
executor, worker streams and communication thread; a broadcast is a
device-to-device copy from the root's buffer (no kernels waiting on one
another, so this is safe on a single GPU).  Every rank's gathered output must
equal the single-GPU echelonize and the oracle bit for bit.  The NCCL
communicator itself is exercised at world 1.
"""
import threading

import numpy as np
import pytest

import oracle
from oracle import restate as R

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    from paper_1806_04211_b200 import gfrref
    gfrref.lib()
    return gfrref


def run_ranks(G, comms, fn):
    outs, errs = [None] * len(comms), []

    def body(r):
        try:
            outs[r] = fn(comms[r])
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=body, args=(r,)) for r in range(len(comms))]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    return outs


def same_output(out, ref, a, b, with_transform=True):
    assert out.rank == ref.rank
    assert [s.members for s in out.upsilon] == [s.members for s in ref.upsilon]
    assert [s.members for s in out.varrho] == [s.members for s in ref.varrho]
    for j in range(b):
        for l in range(j, b):
            assert out.block(0, j, l) == ref.block(0, j, l), ("R", j, l)
    if with_transform:
        for j in range(b):
            for h in range(a):
                assert out.block(1, j, h) == ref.block(1, j, h), ("TM", j, h)
        for i in range(a):
            for h in range(i + 1):
                assert out.block(2, i, h) == ref.block(2, i, h), ("TK", i, h)


@pytest.mark.parametrize("world", [1, 2, 3, 4])
@pytest.mark.parametrize("p,m,n,block,kind", [
    (3, 120, 120, 30, "random"), (2, 256, 192, 64, "random"), (7, 150, 130, 40, "product"),
    (251, 96, 128, 32, "random"),
])
def test_loopback_ranks_match_single_gpu(G, world, p, m, n, block, kind):
    f = G.FieldSpec(p)
    C = G.random_matrix(f, m, n, 11) if kind == "random" else G.random_product_matrix(f, m, n, 37, 11)
    opts = G.EchelonizeOptions(block=block, threads=2)
    ref = G.echelonize(C, f, opts)
    comms = G.Comm.loopback(world)
    outs = run_ranks(G, comms, lambda c: G.echelonize_dist(c, f, m, n, opts, C=C))
    a, b = len(ref.chop.row_parts), len(ref.chop.col_parts)
    for out in outs:
        same_output(out, ref, a, b)


def test_loopback_generated_inputs_and_no_transform(G):
    p, m, n, block, seed = 2, 512, 512, 128, 5
    f = G.FieldSpec(p)
    want = R.blocked_from_oracle(p, oracle.random_matrix(p, m, n, seed), block)
    comms = G.Comm.loopback(4)
    outs = run_ranks(G, comms, lambda c: G.echelonize_dist(c, f, m, n, G.EchelonizeOptions(block=block, threads=2),
                                                           seed=seed))
    for out in outs:
        assert out.rank == want.rank
        assert [s.members for s in out.upsilon] == [s.members for s in want.upsilon]
        np.testing.assert_array_equal(out.materialize_transform().numpy(), want.materialize_transform())
    lean = run_ranks(G, G.Comm.loopback(2),
                     lambda c: G.echelonize_dist(c, f, m, n, G.EchelonizeOptions(block=block, with_transform=False),
                                                 seed=seed))
    for out in lean:
        assert out.rank == want.rank
        np.testing.assert_array_equal(out.assembled_R().numpy(), want.assembled_R())


def test_nccl_world_one(G):
    """The NCCL communicator path (ncclCommInitRank / ncclBroadcast) with a
    single rank: broadcasts are local, the executor is the sharded one."""
    p, m, n, block = 3, 200, 200, 50
    f = G.FieldSpec(p)
    C = G.random_matrix(f, m, n, 3)
    comm = G.Comm.nccl(1, 0, G.Comm.nccl_unique_id())
    out = G.echelonize_dist(comm, f, m, n, G.EchelonizeOptions(block=block, threads=2), C=C)
    ref = G.echelonize(C, f, G.EchelonizeOptions(block=block))
    same_output(out, ref, 4, 4)
