"""TEST INFRASTRUCTURE ONLY -- numpy restatement of the reference's block jobs,
composite tasks and Chief plan, used as the task-level checker.

Matrices are numpy uint8 arrays (shape carries zero-dimensional cases),
index sets are ``IndexSet(universe, members)`` and bit strings are tuples of
0/1.  Every function cites the reference file:line it restates.  Products go
through the C restatement ``oracle.mad``; single-block elimination through
``oracle.oracle_rref`` (the reference's ``ech`` and ``oracle_rref`` agree on
all five outputs -- canonical ECH, pinned in tests/test_oracle.py).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import mad as _mad, oracle_rref as _oracle_rref


# ------------------------------------------------------------------ value types
@dataclass(frozen=True)
class IndexSet:
    """reference include/gfrref/matrix.hpp:53-70"""
    universe: int
    members: tuple = ()

    def __post_init__(self):
        mem = tuple(int(v) for v in self.members)
        for q, v in enumerate(mem):
            if v >= self.universe:
                raise ValueError("index set: member out of universe")
            if q and v <= mem[q - 1]:
                raise ValueError("index set: members must be increasing")
        object.__setattr__(self, "members", mem)

    def __len__(self):
        return len(self.members)


def complement(s: IndexSet) -> IndexSet:
    """reference src/matrix.cpp:50-63"""
    mem = set(s.members)
    return IndexSet(s.universe, tuple(v for v in range(s.universe) if v not in mem))


def zeros(r, c):
    return np.zeros((r, c), np.uint8)


# ------------------------------------------------------------------ jobs
def mul(p, b, c):
    """reference src/jobs.cpp:193-195"""
    return _mad(p, b, c)


def mad(p, a, b, c):
    """reference src/jobs.cpp:197-200"""
    return _mad(p, b, c, a)


def take_rows(m, rows):
    """reference src/matrix.cpp:156-165"""
    return np.ascontiguousarray(m[list(rows), :]) if len(rows) else zeros(0, m.shape[1])


def take_cols(m, cols):
    """reference src/matrix.cpp:167-176"""
    return np.ascontiguousarray(m[:, list(cols)]) if len(cols) else zeros(m.shape[0], 0)


def cex(h, gamma: IndexSet):
    """reference src/jobs.cpp:227-232"""
    if gamma.universe != h.shape[1]:
        raise ValueError("cex: universe mismatch")
    return take_cols(h, gamma.members), take_cols(h, complement(gamma).members)


def rex(h, rho: IndexSet):
    """reference src/jobs.cpp:234-239"""
    if rho.universe != h.shape[0]:
        raise ValueError("rex: universe mismatch")
    return take_rows(h, rho.members), take_rows(h, complement(rho).members)


def unh(rho1: IndexSet, rho2: IndexSet):
    """reference src/jobs.cpp:241-264"""
    comp = complement(rho1)
    if rho2.universe != len(comp):
        raise ValueError("unh: universe of rho2 must be the complement size")
    emb = [comp.members[i] for i in rho2.members]
    merged, u = [], []
    i = j = 0
    while i < len(rho1) or j < len(emb):
        if j >= len(emb) or (i < len(rho1) and rho1.members[i] < emb[j]):
            merged.append(rho1.members[i]); u.append(0); i += 1
        else:
            merged.append(emb[j]); u.append(1); j += 1
    return IndexSet(rho1.universe, tuple(merged)), tuple(u)


def un0(rho2: IndexSet):
    """reference src/jobs.cpp:266-270"""
    return rho2, tuple([1] * len(rho2))


def mkr(rho1: IndexSet, rho2: IndexSet):
    """reference src/jobs.cpp:272-285"""
    out = [0] * len(rho2)
    i = 0
    for l, v in enumerate(rho2.members):
        if i < len(rho1) and rho1.members[i] == v:
            out[l] = 1
            i += 1
    if i != len(rho1):
        raise ValueError("mkr: rho1 must be a subset of rho2")
    return tuple(out)


def rrf(u, b, c):
    """reference src/jobs.cpp:287-301"""
    zeros_ = sum(1 for x in u if not x)
    if zeros_ != b.shape[0] or len(u) - zeros_ != c.shape[0]:
        raise ValueError("rrf: bit counts do not match row counts")
    if b.shape[1] != c.shape[1] and b.shape[0] != 0 and c.shape[0] != 0:
        raise ValueError("rrf: column counts disagree")
    cols = b.shape[1] if (b.shape[0] != 0 or c.shape[0] == 0) else c.shape[1]
    out = zeros(len(u), cols)
    bi = ci = 0
    for l, bit in enumerate(u):
        if bit:
            out[l] = c[ci]; ci += 1
        else:
            out[l] = b[bi]; bi += 1
    return out


def crz(m, lam, out_cols):
    """reference src/jobs.cpp:303-316"""
    if len(lam) != out_cols:
        raise ValueError("crz: lambda length must equal out_cols")
    if sum(lam) != m.shape[1]:
        raise ValueError("crz: ones count must equal input columns")
    out = zeros(m.shape[0], out_cols)
    src = 0
    for l, bit in enumerate(lam):
        if bit:
            out[:, l] = m[:, src]
            src += 1
    return out


def adi(k, delta):
    """reference src/jobs.cpp:318-331"""
    if len(delta) != k.shape[1]:
        raise ValueError("adi: delta length must equal columns")
    if sum(delta) > k.shape[0]:
        raise ValueError("adi: more marked positions than rows")
    out = k.copy()
    i = 0
    for l, bit in enumerate(delta):
        if bit:
            out[i, l] = 1
            i += 1
    return out


@dataclass
class EchResult:
    """reference include/gfrref/jobs.hpp:20-32"""
    M: np.ndarray
    K: np.ndarray
    R: np.ndarray
    rho: IndexSet
    gamma: IndexSet

    def rank(self):
        return len(self.gamma)


def ech(p, h) -> EchResult:
    """reference src/jobs.cpp:202-225 -- canonical, so computed with the
    sequential oracle (src/chief.cpp:427-487)."""
    a, b = h.shape
    o = _oracle_rref(p, h)
    return EchResult(o["M"], o["K"], o["R"], IndexSet(a, tuple(o["rho"])), IndexSet(b, tuple(o["gamma"])))


# ------------------------------------------------------------------ packages
@dataclass
class PkgA:
    """reference include/gfrref/packages.hpp:17-26"""
    M: np.ndarray
    K: np.ndarray
    rho_prime: IndexSet
    A: np.ndarray | None = None
    E: np.ndarray | None = None
    lam: tuple | None = None


@dataclass
class PkgD:
    """reference include/gfrref/packages.hpp:30-36"""
    R: np.ndarray = field(default_factory=lambda: zeros(0, 0))
    gamma: IndexSet = field(default_factory=lambda: IndexSet(0, ()))


@dataclass
class PkgE:
    """reference include/gfrref/packages.hpp:40-45"""
    rho: IndexSet
    delta: tuple


# ------------------------------------------------------------------ tasks
def clear_down(p, C, D: PkgD, i):
    """reference src/tasks.cpp:15-46"""
    if i == 0:
        e = ech(p, C)
        return PkgD(e.R, e.gamma), PkgA(e.M, e.K, e.rho)
    if D.gamma.universe != C.shape[1]:
        raise ValueError("clear_down: column state universe mismatch")
    a_cols, c_rest = cex(C, D.gamma)
    h = mad(p, c_rest, a_cols, D.R)
    e = ech(p, h)
    e_mid, r_old = cex(D.R, e.gamma)
    r_upd = mad(p, r_old, e_mid, e.R)
    gam, lam = unh(D.gamma, e.gamma)
    return PkgD(rrf(lam, r_upd, e.R), gam), PkgA(e.M, e.K, e.rho, a_cols, e_mid, lam)


def update_row(p, A: PkgA, C, B, i):
    """reference src/tasks.cpp:48-68"""
    if (i == 0) == (B is not None):
        raise ValueError("update_row: B must be given iff i > 0")
    z = C if i == 0 else mad(p, C, A.A, B)
    v, w = rex(z, A.rho_prime)
    x = mul(p, A.M, v)
    b_out = x if i == 0 else rrf(A.lam, mad(p, B, A.E, x), x)
    return mad(p, w, A.K, v), b_out


def update_row_trafo(p, A: PkgA, K, M, E: PkgE, i, h, j):
    """reference src/tasks.cpp:70-123"""
    if h > i:
        raise ValueError("update_row_trafo: h must be <= i")
    if (j == 0) == (K is not None):
        raise ValueError("update_row_trafo: K must be given iff j > 0")
    if (h == i) == (M is not None):
        raise ValueError("update_row_trafo: M must be given iff h < i")
    kx = None
    if j > 0:
        kx = crz(K, tuple(b ^ 1 for b in E.delta), len(E.delta))
    if h == i and j == 0:
        m_out = A.M
        if i != 0:
            m_out = rrf(A.lam, mul(p, A.E, m_out), m_out)
        return A.K, m_out
    if h != i:
        if A.A is None:
            raise ValueError("update_row_trafo: package lacks A")
        z = mad(p, kx, A.A, M) if j > 0 else mul(p, A.A, M)
    else:
        z = kx
    v, w = rex(z, A.rho_prime)
    if h == i:
        v = adi(v, E.delta)
    x = mul(p, A.M, v)
    if h == i and i == 0:
        m_out = x
    else:
        s = mad(p, M, A.E, x) if h != i else mul(p, A.E, x)
        m_out = rrf(A.lam, s, x)
    return mad(p, w, A.K, v), m_out


def extend(A: PkgA, E: PkgE | None, j):
    """reference src/tasks.cpp:125-139"""
    if (j == 0) == (E is not None):
        raise ValueError("extend: E must be given iff j > 0")
    rho, delta = un0(A.rho_prime) if j == 0 else unh(E.rho, A.rho_prime)
    return PkgE(rho, delta)


def row_lengthen(M, E1: PkgE, E2: PkgE):
    """reference src/tasks.cpp:141-144"""
    marks = mkr(E1.rho, E2.rho)
    return crz(M, marks, len(marks))


def pre_clear_up(B, D: PkgD):
    """reference src/tasks.cpp:146-148"""
    return cex(B, D.gamma)


def clear_up(p, R, X, M):
    """reference src/tasks.cpp:150-153"""
    return mad(p, R, X, M)


def copy_d(D: PkgD):
    """reference src/tasks.cpp:155"""
    return D.R


# ------------------------------------------------------------------ chief
def chop_axis(total, block, remainder_first=False):
    """reference src/chief.cpp:33-42"""
    full, rem = divmod(total, block)
    parts = []
    if rem and remainder_first:
        parts.append(rem)
    parts += [block] * full
    if rem and not remainder_first:
        parts.append(rem)
    return parts


def chop(m, n, block, remainder_first=False):
    """reference src/chief.cpp:46-53"""
    if block < 1:
        raise ValueError("chop: block must be >= 1")
    return chop_axis(m, block, remainder_first), chop_axis(n, block, remainder_first)


@dataclass
class Output:
    """Mirror of reference ``EchelonOutput`` (include/gfrref/chief.hpp:33-59)."""
    p: int
    row_parts: list
    col_parts: list
    rank: int
    upsilon: list
    varrho: list
    R_blocks: dict
    T_M_blocks: dict
    T_K_blocks: dict
    with_transform: bool = True

    def row_offset(self, i):
        return sum(self.row_parts[:i])

    def col_offset(self, j):
        return sum(self.col_parts[:j])

    def global_upsilon(self):
        """reference src/chief.cpp:388-396"""
        return [self.col_offset(j) + v for j, s in enumerate(self.upsilon) for v in s.members]

    def global_varrho(self):
        """reference src/chief.cpp:398-406"""
        return [self.row_offset(i) + v for i, s in enumerate(self.varrho) for v in s.members]

    def assembled_R(self):
        """reference src/chief.cpp:408-425"""
        n = sum(self.col_parts)
        out = zeros(self.rank, n - self.rank)
        row = 0
        b = len(self.col_parts)
        for j in range(b):
            for t in range(len(self.upsilon[j])):
                col = 0
                for l in range(b):
                    width = self.col_parts[l] - len(self.upsilon[l])
                    if l >= j and width:
                        out[row, col:col + width] = self.R_blocks[(j, l)][t]
                    col += width
                row += 1
        return out

    def materialize_transform(self):
        """reference src/chief.cpp:489-520"""
        m = sum(self.row_parts)
        a, b = len(self.row_parts), len(self.col_parts)
        t = zeros(m, m)
        row = 0
        for j in range(b):
            for q in range(len(self.upsilon[j])):
                for h in range(a):
                    off = self.row_offset(h)
                    mjh = self.T_M_blocks[(j, h)]
                    for s, v in enumerate(self.varrho[h].members):
                        t[row, off + v] = mjh[q, s]
                row += 1
        for i in range(a):
            off = self.row_offset(i)
            rest = complement(self.varrho[i])
            for u, v in enumerate(rest.members):
                t[row, off + v] = 1
                for h in range(i + 1):
                    hoff = self.row_offset(h)
                    kih = self.T_K_blocks[(i, h)]
                    for s, w in enumerate(self.varrho[h].members):
                        t[row, hoff + w] = kih[u, s]
                row += 1
        return t


def echelonize(p, C, block, with_transform=True, remainder_first=False) -> Output:
    """Sequential restatement of reference ``build_plan`` + ``run`` +
    ``echelonize`` (src/chief.cpp:67-386): tasks run in the plan's insertion
    order, which is a topological order of its slot graph."""
    m, n = C.shape
    rp, cp = chop(m, n, block, remainder_first)
    a, b = len(rp), len(cp)
    ro = np.cumsum([0] + rp)
    co = np.cumsum([0] + cp)
    if a == 0 or b == 0:
        return Output(p, rp, cp, 0, [IndexSet(c, ()) for c in cp], [IndexSet(r, ()) for r in rp],
                      {(j, l): zeros(0, cp[l]) for j in range(b) for l in range(j, b)},
                      {}, {(i, h): zeros(rp[i], 0) for i in range(a) for h in range(i + 1)}, with_transform)
    Cs = {(i, k, 0): np.ascontiguousarray(C[ro[i]:ro[i + 1], co[k]:co[k + 1]]) for i in range(a) for k in range(b)}
    D, A, B, E, K, M, R, X = {}, {}, {}, {}, {}, {}, {}, {}
    # Step 1 (src/chief.cpp:114-180)
    for j in range(b):
        for i in range(a):
            D[(j, i)], A[(i, j)] = clear_down(p, Cs[(i, j, j)], D[(j, i - 1)] if i > 0 else PkgD(), i)
            E[(i, j)] = extend(A[(i, j)], E[(i, j - 1)] if j > 0 else None, j)
            for k in range(j + 1, b):
                Cs[(i, k, j + 1)], B[(j, k, i)] = update_row(
                    p, A[(i, j)], Cs[(i, k, j)], B[(j, k, i - 1)] if i > 0 else None, i)
            if with_transform:
                for h in range(i + 1):
                    K[(i, h, j)], M[(j, h, i - h)] = update_row_trafo(
                        p, A[(i, j)], K[(i, h, j - 1)] if j > 0 else None,
                        M[(j, h, i - 1 - h)] if h < i else None, E[(h, j)], i, h, j)
    # Step 2 (src/chief.cpp:182-199)
    if with_transform:
        for j in range(b):
            for h in range(a):
                M[(j, h, a - h)] = row_lengthen(M[(j, h, a - 1 - h)], E[(h, j)], E[(h, b - 1)])
    # Step 3 (src/chief.cpp:203-262)
    for k in range(b):
        R[(k, k, 0)] = copy_d(D[(k, a - 1)])
    for k in range(b - 1, 0, -1):
        for j in range(k):
            X[(j, k)], R[(j, k, 0)] = pre_clear_up(B[(j, k, a - 1)], D[(k, a - 1)])
            for l in range(k, b):
                R[(j, l, l - k + 1)] = clear_up(p, R[(j, l, l - k)], X[(j, k)], R[(k, l, l - k)])
            if with_transform:
                for h in range(a):
                    M[(j, h, a - h + (b - k))] = clear_up(p, M[(j, h, a - h + (b - 1 - k))], X[(j, k)],
                                                          M[(k, h, a - h + (b - 1 - k))])
    ups = [D[(j, a - 1)].gamma for j in range(b)]
    return Output(
        p, rp, cp, sum(len(g) for g in ups), ups, [E[(i, b - 1)].rho for i in range(a)],
        {(j, l): R[(j, l, l - j)] for j in range(b) for l in range(j, b)},
        {(j, h): M[(j, h, a - h + (b - 1 - j))] for j in range(b) for h in range(a)} if with_transform else {},
        {(i, h): K[(i, h, b - 1)] for i in range(a) for h in range(i + 1)} if with_transform else {},
        with_transform)


def blocked_from_oracle(p, C, block, remainder_first=False) -> Output:
    """Block-level outputs derived from the global sequential oracle.

    The outputs are canonical: each block of the reference's
    EchelonOutput is a slice of the global (rank, Upsilon, varrho, R, T)
    computed by ``oracle_rref`` -- T_M_blocks[j][h] = M rows of the pivots in
    block column j restricted to the selected rows of block row h, etc.
    """
    m, n = C.shape
    rp, cp = chop(m, n, block, remainder_first)
    a, b = len(rp), len(cp)
    o = _oracle_rref(p, C)
    r = o["rank"]
    gam = [int(v) for v in o["gamma"]]
    rho = [int(v) for v in o["rho"]]
    ro = np.cumsum([0] + rp)
    co = np.cumsum([0] + cp)
    ups = [IndexSet(cp[j], tuple(v - co[j] for v in gam if co[j] <= v < co[j + 1])) for j in range(b)]
    vrh = [IndexSet(rp[i], tuple(v - ro[i] for v in rho if ro[i] <= v < ro[i + 1])) for i in range(a)]
    gset = set(gam)
    nonpiv = [c for c in range(n) if c not in gset]
    piv_block = [next(j for j in range(b) if co[j] <= v < co[j + 1]) for v in gam]
    Rb = {}
    for j in range(b):
        rows = [q for q in range(r) if piv_block[q] == j]
        for l in range(j, b):
            cols = [t for t, c in enumerate(nonpiv) if co[l] <= c < co[l + 1]]
            Rb[(j, l)] = np.ascontiguousarray(o["R"][np.ix_(rows, cols)]) if rows and cols else zeros(len(rows), len(cols))
    TM, TK = {}, {}
    rho_pos = {v: s for s, v in enumerate(rho)}
    for j in range(b):
        rows = [q for q in range(r) if piv_block[q] == j]
        for h in range(a):
            cols = [rho_pos[ro[h] + v] for v in vrh[h].members]
            TM[(j, h)] = np.ascontiguousarray(o["M"][np.ix_(rows, cols)]) if rows and cols else zeros(len(rows), len(cols))
    nonsel = [t for t in range(m) if t not in rho_pos]
    for i in range(a):
        rows = [u for u, t in enumerate(nonsel) if ro[i] <= t < ro[i + 1]]
        for h in range(i + 1):
            cols = [rho_pos[ro[h] + v] for v in vrh[h].members]
            TK[(i, h)] = np.ascontiguousarray(o["K"][np.ix_(rows, cols)]) if rows and cols else zeros(len(rows), len(cols))
    return Output(p, rp, cp, r, ups, vrh, Rb, TM, TK, True)
