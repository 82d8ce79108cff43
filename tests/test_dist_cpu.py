"""CPU (gloo, world_size >= 2) test of the sharded Chief's dataflow.

The product's ownership map and broadcast schedule (gfq_dist_plan, host-only
C ABI) are executed rank by rank with the numpy restatement of the
reference tasks (oracle/restate.py) and torch.distributed gloo broadcasts in
the schedule order -- exactly the contract of the CUDA/NCCL executor
(csrc/host/dist.cpp): every task runs on its owner, the only packages that
cross ranks are PkgA(i,j) and X(j,k), and issuing the broadcasts in the
fixed order never deadlocks.  Each rank's owned output blocks are gathered
to rank 0 and compared with the single-process Chief.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from oracle import restate as R

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def sharded_run(p, C, block, with_transform, world, rank, owner, sched):
    """restate.echelonize's loops, executing only owned tasks; PkgA / X come
    from broadcasts performed lazily in schedule order."""
    m, n = C.shape
    rp, cp = R.chop(m, n, block)
    a, b = len(rp), len(cp)
    ro = np.cumsum([0] + rp)
    co = np.cumsum([0] + cp)
    Cs = {(i, k, 0): np.ascontiguousarray(C[ro[i]:ro[i + 1], co[k]:co[k + 1]])
          for i in range(a) for k in range(b) if k % world == rank}
    D, A, B, E, K, M, Rr, X = {}, {}, {}, {}, {}, {}, {}, {}
    pos = {("A", it[1], it[2]) if it[0] else ("X", it[2], it[3]): q for q, it in enumerate(sched)}
    done = [0]  # number of schedule items performed

    def perform_through(t):
        while done[0] <= t:
            is_a, i, j, k, root = sched[done[0]]
            store, key = (A, (i, j)) if is_a else (X, (j, k))
            obj = [store.get(key) if rank == root else None]
            assert rank != root or obj[0] is not None, "root has not produced its package"
            dist.broadcast_object_list(obj, src=root)
            store[key] = obj[0]
            done[0] += 1

    def need(kind, x, y):
        perform_through(pos[(kind, x, y)])

    def mine(kind, c0, c1, c2):
        o = owner[(kind, c0, c1, c2)]
        return o == -1 or o == rank

    # Step 1 in the schedule's PkgA order (the wavefront: i + j, then j) --
    # a valid sequential order of the plan, and the order the broadcasts need
    a_order = [(it[1], it[2]) for it in sched if it[0]]
    assert sorted(a_order) == [(i, j) for i in range(a) for j in range(b)]
    for (i, j) in a_order:
        if mine("ClearDown", i, j, -1):
            D[(j, i)], A[(i, j)] = R.clear_down(p, Cs[(i, j, j)], D[(j, i - 1)] if i > 0 else R.PkgD(), i)
        need("A", i, j)
        E[(i, j)] = R.extend(A[(i, j)], E[(i, j - 1)] if j > 0 else None, j)
        for k in range(j + 1, b):
            if mine("UpdateRow", i, j, k):
                Cs[(i, k, j + 1)], B[(j, k, i)] = R.update_row(
                    p, A[(i, j)], Cs[(i, k, j)], B[(j, k, i - 1)] if i > 0 else None, i)
        if with_transform:
            for h in range(i + 1):
                if mine("UpdateRowTrafo", i, j, h):
                    K[(i, h, j)], M[(j, h, i - h)] = R.update_row_trafo(
                        p, A[(i, j)], K[(i, h, j - 1)] if j > 0 else None,
                        M[(j, h, i - 1 - h)] if h < i else None, E[(h, j)], i, h, j)
    if with_transform:
        for j in range(b):
            for h in range(a):
                if mine("RowLengthen", -1, j, h):
                    M[(j, h, a - h)] = R.row_lengthen(M[(j, h, a - 1 - h)], E[(h, j)], E[(h, b - 1)])
    for k in range(b):
        if mine("Copy", -1, k, -1):
            Rr[(k, k, 0)] = R.copy_d(D[(k, a - 1)])
    for k in range(b - 1, 0, -1):
        for j in range(k):
            if mine("PreClearUp", -1, j, k):
                X[(j, k)], Rr[(j, k, 0)] = R.pre_clear_up(B[(j, k, a - 1)], D[(k, a - 1)])
            need("X", j, k)
            for l in range(k, b):
                if mine("ClearUp", k, j, l) and l % world == rank:
                    Rr[(j, l, l - k + 1)] = R.clear_up(p, Rr[(j, l, l - k)], X[(j, k)], Rr[(k, l, l - k)])
            if with_transform:
                for h in range(a):
                    if h % world == rank:
                        M[(j, h, a - h + (b - k))] = R.clear_up(
                            p, M[(j, h, a - h + (b - 1 - k))], X[(j, k)], M[(k, h, a - h + (b - 1 - k))])
    perform_through(len(sched) - 1)
    # owned final blocks
    out = {"ups": {j: D[(j, a - 1)].gamma for j in range(b) if j % world == rank},
           "rho": {i: E[(i, b - 1)].rho for i in range(a)},
           "R": {(j, l): Rr[(j, l, l - j)] for j in range(b) for l in range(j, b) if l % world == rank}}
    if with_transform:
        out["TM"] = {(j, h): M[(j, h, a - h + (b - 1 - j))] for j in range(b) for h in range(a) if h % world == rank}
        out["TK"] = {(i, h): K[(i, h, b - 1)] for i in range(a) for h in range(i + 1) if h % world == rank}
    return out


def test_broadcast_order_is_wavefront():
    """PkgA broadcasts follow the Step-1 wavefront (anti-diagonal i + j, then
    j) and precede every X broadcast; X in Step-3 order (k descending)."""
    import sys
    sys.path.insert(0, ROOT)
    from paper_1806_04211_b200 import gfrref as G
    _, sched = G.dist_plan(40, 48, 8, True, 4)
    a_items = [(it[1], it[2]) for it in sched if it[0]]
    assert a_items == sorted(a_items, key=lambda ij: (ij[0] + ij[1], ij[1]))
    first_x = next(q for q, it in enumerate(sched) if not it[0])
    assert all(it[0] for it in sched[:first_x]) and not any(it[0] for it in sched[first_x:])
    ks = [it[3] for it in sched[first_x:]]
    assert ks == sorted(ks, reverse=True)


def _worker(rank, world, port, case, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    dist.init_process_group("gloo", rank=rank, world_size=world, init_method=f"tcp://127.0.0.1:{port}")
    try:
        import sys
        sys.path.insert(0, ROOT)
        from paper_1806_04211_b200 import gfrref as G
        p, m, n, block, wt, kind = case
        C = oracle.random_matrix(p, m, n, 7) if kind == "random" else \
            oracle.random_product_matrix(p, m, n, min(m, n) // 2, 7)
        nodes, sched = G.dist_plan(m, n, block, wt, world)
        owner = {}
        for (kname, c0, c1, c2, o) in nodes:
            owner[(kname, c0, c1, c2)] = o
        # every cross-rank consumer input is covered by the schedule
        assert all(it[4] == (it[2] if it[0] else it[3]) % world for it in sched)
        out = sharded_run(p, C, block, wt, world, rank, owner, sched)
        gathered = [None] * world
        dist.all_gather_object(gathered, out)
        if rank == 0:
            want = R.echelonize(p, C, block, wt)
            ups, Rb, TM, TK = {}, {}, {}, {}
            for o in gathered:
                ups.update(o["ups"])
                Rb.update(o["R"])
                TM.update(o.get("TM", {}))
                TK.update(o.get("TK", {}))
            ok = all(ups[j] == want.upsilon[j] for j in range(len(want.col_parts)))
            ok &= all(gathered[0]["rho"][i] == want.varrho[i] for i in range(len(want.row_parts)))
            ok &= all(np.array_equal(Rb[key], want.R_blocks[key]) for key in want.R_blocks)
            if wt:
                ok &= all(np.array_equal(TM[key], want.T_M_blocks[key]) for key in want.T_M_blocks)
                ok &= all(np.array_equal(TK[key], want.T_K_blocks[key]) for key in want.T_K_blocks)
            q.put(bool(ok))
    except Exception as e:  # surface the failure to the parent
        if rank == 0:
            q.put(repr(e))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case,world", [
    ((3, 12, 12, 3, True, "random"), 2),
    ((2, 20, 16, 4, True, "random"), 2),
    ((5, 18, 21, 4, True, "product"), 2),
    ((7, 15, 15, 4, False, "random"), 2),
    ((3, 16, 16, 3, True, "product"), 3),
    ((2, 24, 20, 4, True, "random"), 4),
    ((3, 22, 26, 5, True, "product"), 4),
])
def test_sharded_chief_gloo(case, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=240)
    res = q.get(timeout=5)
    assert res is True, res
    assert all(pr.exitcode == 0 for pr in procs)
