"""Python mirror of the reference ``gfrref`` API over the B200 C ABI.

Same names, argument meaning and error behaviour as the reference's C++
headers (include/gfrref/{field,matrix,jobs,packages,tasks,chief}.hpp), so
the parity tests read like the reference's own tests:

    f = FieldSpec(3)
    e = ech(f, mat_build(3, 3, [[0, 2, 2], [0, 2, 2], [1, 0, 1]]))
    assert e.M == mat_build(2, 2, [[0, 2], [1, 0]])

Matrices are device-resident (``Matrix`` wraps a ``gfq_mat`` handle in HBM);
index sets and bit strings are small host values.  Shape errors raise
``ValueError`` (the reference's ``std::invalid_argument``) with the
reference's message text.  Every compute call goes through libgfq.so; there
is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _capi

_lib = None


class GfqError(RuntimeError):
    code = -1


class CudaError(GfqError):
    code = 3


class TaskError(GfqError):
    code = 2


class LogicError(GfqError):
    code = 4


def default_device() -> int:
    """GFQ_DEVICE, else the launcher's LOCAL_RANK (one process per GPU), else 0."""
    for var in ("GFQ_DEVICE", "LOCAL_RANK"):
        if os.environ.get(var, "").strip().isdigit():
            return int(os.environ[var])
    return 0


def lib():
    """The loaded libgfq.so, initialised on default_device() (the library's
    CUDA runtime is its own: its current device is set here, not by torch)."""
    global _lib
    if _lib is None:
        l = _capi.load()
        rc = l.gfq_init(default_device())
        if rc != 0:
            raise CudaError(l.gfq_last_error().decode())
        _lib = l
    return _lib


_raw = None


def raw_lib():
    """libgfq.so without device initialisation (host-only entry points)."""
    global _raw
    if _raw is None:
        _raw = _capi.load()
    return _raw


def _check(rc):
    if rc == 0:
        return
    msg = (_lib or raw_lib()).gfq_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    if rc == 5:
        raise ZeroDivisionError(msg)
    if rc == 3:
        raise CudaError(msg)
    if rc == 4:
        raise LogicError(msg)
    raise TaskError(msg)


def _vp():
    return ctypes.c_void_p()


# ---------------------------------------------------------------- values
class FieldSpec:
    """GF(p) or GF(p^k) (reference include/gfrref/field.hpp:20-110).

    ``FieldSpec(p)`` is the prime field (p < 2**16);
    ``FieldSpec(p, k, modulus=None)`` the extension field with a monic
    irreducible modulus ``[c0, ..., ck]`` (None: the reference's default,
    the lexicographically first one), p**k < 2**20.  Elements are encoded
    like the reference, ``sum_i c_i p**i``: one byte each for p <= 251 /
    p**k <= 256 (the tensor-core path), u32 for the "wide" rest.  ``code`` is
    the integer the C ABI takes as its field argument (p for a prime field).
    """

    def __init__(self, p: int, k: int = 1, modulus=None):
        p, k = int(p), int(k)
        if k == 1 and modulus is None:
            if p < 2 or any(p % d == 0 for d in range(2, int(p ** 0.5) + 1)):
                raise ValueError("field: p must be prime")
            if p >= 1 << 16:
                raise ValueError("field: p must be < 2^16")
            self.p, self.k, self.q, self.code = p, 1, p, p
            self.modulus = (0, 1)
            return
        code = ctypes.c_uint32()
        mod = None if modulus is None else (ctypes.c_uint32 * len(modulus))(*[int(c) for c in modulus])
        _check(raw_lib().gfq_field_register(p, k, mod, 0 if modulus is None else len(modulus), ctypes.byref(code)))
        self._from_code(code.value)

    def _from_code(self, code: int):
        p, k, q = ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_uint32()
        mod = (ctypes.c_uint32 * 32)()
        _check(raw_lib().gfq_field_info(code, ctypes.byref(p), ctypes.byref(k), ctypes.byref(q), mod))
        self.p, self.k, self.q, self.code = p.value, k.value, q.value, code
        self.modulus = tuple(mod[i] for i in range(self.k + 1))

    @classmethod
    def from_code(cls, code: int) -> "FieldSpec":
        f = cls.__new__(cls)
        f._from_code(int(code))
        return f

    def order(self):
        return self.q

    @property
    def wide(self) -> bool:
        """u32 element storage (p > 251, or p**k > 256)"""
        return self.q > 256 if self.k > 1 else self.p > 251

    @property
    def esize(self) -> int:
        return 4 if self.wide else 1

    def _op(self, op, a, b=0):
        out = ctypes.c_uint32()
        _check(raw_lib().gfq_field_op(self.code, op, int(a), int(b), ctypes.byref(out)))
        return out.value

    def add(self, a, b):
        return self._op(0, a, b)

    def mul(self, a, b):
        return self._op(1, a, b)

    def neg(self, a):
        return self._op(2, a)

    def inv(self, a):
        return self._op(3, a)

    def __eq__(self, o):
        return isinstance(o, FieldSpec) and (o.p, o.k, o.modulus) == (self.p, self.k, self.modulus)

    def __hash__(self):
        return hash((self.p, self.k, self.modulus))

    def __repr__(self):
        return f"GF({self.p})" if self.k == 1 else f"GF({self.p}^{self.k})"


def default_modulus(p: int, k: int):
    """Reference default_modulus (include/gfrref/field.hpp:118)."""
    out = (ctypes.c_uint32 * (int(k) + 1))()
    _check(raw_lib().gfq_default_modulus(int(p), int(k), out))
    return list(out)


class Matrix:
    """Device-resident dense u8 matrix (reference Matrix, include/gfrref/matrix.hpp:15-43)."""

    __slots__ = ("h", "rows", "cols", "esize")

    def __init__(self, handle, rows=None, cols=None, esize=None):
        self.h = handle
        if rows is None:
            r, c = ctypes.c_int64(), ctypes.c_int64()
            _check(lib().gfq_mat_shape(handle, ctypes.byref(r), ctypes.byref(c)))
            rows, cols = r.value, c.value
        self.rows, self.cols = int(rows), int(cols)
        if esize is None:
            e = ctypes.c_int()
            _check(lib().gfq_mat_esize(handle, ctypes.byref(e)))
            esize = e.value
        self.esize = int(esize)

    def __del__(self):
        if self.h and _lib is not None:
            _lib.gfq_mat_free(self.h)
            self.h = None

    @staticmethod
    def from_numpy(a, esize=None) -> "Matrix":
        """u8 storage for uint8 arrays, u32 (wide fields) for wider dtypes or
        esize=4."""
        a = np.asarray(a)
        if esize is None:
            esize = 1 if a.dtype.itemsize == 1 else 4
        if a.ndim != 2:
            raise ValueError("matrix: expected a 2-D array")
        r, c = a.shape
        h = _vp()
        if esize == 4:
            a = np.ascontiguousarray(a.astype(np.uint32))
            src = a if a.size else np.zeros(1, np.uint32)
            _check(lib().gfq_mat_upload32(r, c, src.ctypes.data_as(_capi.c_u32p), max(c, 1), ctypes.byref(h)))
            return Matrix(h, r, c, 4)
        a = np.ascontiguousarray(a.astype(np.uint8))
        src = a if a.size else np.zeros(1, np.uint8)
        _check(lib().gfq_mat_upload(r, c, src.ctypes.data_as(_capi.c_u8p), max(c, 1), ctypes.byref(h)))
        return Matrix(h, r, c, 1)

    @staticmethod
    def zeros(rows: int, cols: int, esize: int = 1) -> "Matrix":
        h = _vp()
        if esize == 4:
            _check(lib().gfq_mat_upload32(rows, cols, None, max(cols, 1), ctypes.byref(h)))
        else:
            _check(lib().gfq_mat_upload(rows, cols, None, max(cols, 1), ctypes.byref(h)))
        return Matrix(h, rows, cols, esize)

    @staticmethod
    def from_device(ptr: int, rows: int, cols: int, ld: int) -> "Matrix":
        h = _vp()
        _check(lib().gfq_mat_copy_device(rows, cols, ctypes.c_void_p(ptr), ld, ctypes.byref(h)))
        return Matrix(h, rows, cols)

    def numpy(self) -> np.ndarray:
        out = np.zeros((self.rows, self.cols), np.uint32 if self.esize == 4 else np.uint8)
        if out.size:
            _check(lib().gfq_mat_download(self.h, out.ctypes.data_as(_capi.c_u8p), self.cols * self.esize))
        return out

    def device_ptr(self):
        p, ld = ctypes.c_void_p(), ctypes.c_int64()
        _check(lib().gfq_mat_device_ptr(self.h, ctypes.byref(p), ctypes.byref(ld)))
        return p.value or 0, ld.value

    @property
    def shape(self):
        return (self.rows, self.cols)

    def at(self, r, c):
        return int(self.numpy()[r, c])

    def __eq__(self, o):
        if isinstance(o, Matrix):
            return self.shape == o.shape and np.array_equal(self.numpy(), o.numpy())
        o = np.asarray(o)
        return self.shape == o.shape and np.array_equal(self.numpy(), o)

    def __repr__(self):
        return f"Matrix({self.rows}x{self.cols}, {self.numpy().tolist()})"


def mat_build(rows: int, cols: int, entries) -> Matrix:
    """reference src/matrix.cpp:15-27"""
    if len(entries) != rows:
        raise ValueError("mat_build: row count mismatch")
    for r in entries:
        if len(r) != cols:
            raise ValueError("mat_build: column count mismatch")
    return Matrix.from_numpy(np.array(entries, np.uint8).reshape(rows, cols))


def mat_eq(a: Matrix, b: Matrix) -> bool:
    return a == b


@dataclass(frozen=True)
class IndexSet:
    """reference include/gfrref/matrix.hpp:53-70"""
    universe: int = 0
    members: tuple = ()

    def __post_init__(self):
        # vectorised checks (the library hands back sets of up to ~10^5
        # members per block; a Python loop cost ~20 ms per echelonize)
        a = np.asarray(self.members, dtype=np.int64).reshape(-1)
        if a.size:
            if int(a.max()) >= self.universe or int(a.min()) < 0:
                raise ValueError("index set: member out of universe")
            if a.size > 1 and bool(np.any(a[1:] <= a[:-1])):
                raise ValueError("index set: members must be increasing")
        object.__setattr__(self, "members", tuple(a.tolist()))

    def __len__(self):
        return len(self.members)

    def size(self):
        return len(self.members)

    def _handle(self):
        arr = np.array(self.members or [0], np.uint32)
        h = _vp()
        _check(lib().gfq_iset_create(self.universe, arr.ctypes.data_as(_capi.c_u32p), len(self.members),
                                     ctypes.byref(h)))
        return h

    @staticmethod
    def _take(h) -> "IndexSet":
        u, n = ctypes.c_uint64(), ctypes.c_uint64()
        _check(lib().gfq_iset_get(h, ctypes.byref(u), ctypes.byref(n), None))
        buf = np.zeros(max(n.value, 1), np.uint32)
        _check(lib().gfq_iset_get(h, None, None, buf.ctypes.data_as(_capi.c_u32p)))
        lib().gfq_iset_free(h)
        return IndexSet(u.value, tuple(int(x) for x in buf[: n.value]))


def index_set_complement(s: IndexSet) -> IndexSet:
    mem = set(s.members)
    return IndexSet(s.universe, tuple(v for v in range(s.universe) if v not in mem))


class BitString(tuple):
    """reference include/gfrref/matrix.hpp:75-87 (a tuple of 0/1)."""

    def __new__(cls, bits: Sequence[int] = ()):
        return super().__new__(cls, (1 if b else 0 for b in bits))

    @property
    def bits(self):
        return tuple(self)

    def count_ones(self):
        return sum(self)

    def count_zeros(self):
        return len(self) - sum(self)

    def _handle(self):
        arr = np.array(list(self) or [0], np.uint8)
        h = _vp()
        _check(lib().gfq_bits_create(arr.ctypes.data_as(_capi.c_u8p), len(self), ctypes.byref(h)))
        return h

    @staticmethod
    def _take(h) -> "BitString":
        n = ctypes.c_uint64()
        _check(lib().gfq_bits_get(h, ctypes.byref(n), None))
        buf = np.zeros(max(n.value, 1), np.uint8)
        _check(lib().gfq_bits_get(h, None, buf.ctypes.data_as(_capi.c_u8p)))
        lib().gfq_bits_free(h)
        return BitString(buf[: n.value].tolist())


class _Temps:
    """Temporary index-set / bit-string handles for one call."""

    def __init__(self):
        self.isets, self.bits = [], []

    def iset(self, s: IndexSet):
        h = s._handle()
        self.isets.append(h)
        return h

    def bit(self, b):
        h = BitString(b)._handle()
        self.bits.append(h)
        return h

    def __enter__(self):
        return self

    def __exit__(self, *a):
        for h in self.isets:
            lib().gfq_iset_free(h)
        for h in self.bits:
            lib().gfq_bits_free(h)


def _mat(h) -> Matrix:
    return Matrix(h)


def _opt_h(m: Optional[Matrix]):
    return m.h if m is not None else None


# ---------------------------------------------------------------- jobs
def _as_matrix(x, f: "FieldSpec" = None) -> Matrix:
    """A device Matrix as is; a host array uploaded (u32 for a wide field f)."""
    if isinstance(x, Matrix):
        return x
    return Matrix.from_numpy(x, f.esize if f is not None else None)


def cpy(a: Matrix) -> Matrix:
    return rrf(BitString([0] * a.rows), a, Matrix.zeros(0, a.cols, a.esize))


def mul(f: FieldSpec, b, c) -> Matrix:
    """reference jobs.hpp:40 -> K1"""
    b, c = _as_matrix(b, f), _as_matrix(c, f)
    h = _vp()
    _check(lib().gfq_mul(f.code, b.h, c.h, ctypes.byref(h)))
    return _mat(h)


def mad(f: FieldSpec, a, b, c) -> Matrix:
    """reference jobs.hpp:43 -> K1 (a + b.c)"""
    a, b, c = _as_matrix(a, f), _as_matrix(b, f), _as_matrix(c, f)
    h = _vp()
    _check(lib().gfq_mad(f.code, a.h, b.h, c.h, ctypes.byref(h)))
    return _mat(h)


mat_mul = mul


def mat_mul_add(f, a, b, c):
    return mad(f, a, b, c)


@dataclass
class EchResult:
    """reference include/gfrref/jobs.hpp:20-32"""
    M: Matrix
    K: Matrix
    R: Matrix
    rho: IndexSet
    gamma: IndexSet

    def rank(self):
        return len(self.gamma)


def ech(f: FieldSpec, h, threshold: int = 256) -> EchResult:
    """reference jobs.hpp:50 -> K2 base case + K1/K3/K4 combines"""
    h = _as_matrix(h, f)
    M, K, R, rho, gam = _vp(), _vp(), _vp(), _vp(), _vp()
    _check(lib().gfq_ech(f.code, h.h, threshold, *(ctypes.byref(x) for x in (M, K, R, rho, gam))))
    return EchResult(_mat(M), _mat(K), _mat(R), IndexSet._take(rho), IndexSet._take(gam))


def cex(h, gamma: IndexSet):
    h = _as_matrix(h)
    a, b = _vp(), _vp()
    with _Temps() as t:
        _check(lib().gfq_cex(h.h, t.iset(gamma), ctypes.byref(a), ctypes.byref(b)))
    return _mat(a), _mat(b)


def rex(h, rho: IndexSet):
    h = _as_matrix(h)
    a, b = _vp(), _vp()
    with _Temps() as t:
        _check(lib().gfq_rex(h.h, t.iset(rho), ctypes.byref(a), ctypes.byref(b)))
    return _mat(a), _mat(b)


def unh(rho1: IndexSet, rho2: IndexSet):
    r, u = _vp(), _vp()
    with _Temps() as t:
        _check(lib().gfq_unh(t.iset(rho1), t.iset(rho2), ctypes.byref(r), ctypes.byref(u)))
    return IndexSet._take(r), BitString._take(u)


def un0(rho2: IndexSet):
    r, u = _vp(), _vp()
    with _Temps() as t:
        _check(lib().gfq_un0(t.iset(rho2), ctypes.byref(r), ctypes.byref(u)))
    return IndexSet._take(r), BitString._take(u)


def mkr(rho1: IndexSet, rho2: IndexSet) -> BitString:
    u = _vp()
    with _Temps() as t:
        _check(lib().gfq_mkr(t.iset(rho1), t.iset(rho2), ctypes.byref(u)))
    return BitString._take(u)


def rrf(u, b, c) -> Matrix:
    b, c = _as_matrix(b), _as_matrix(c)
    h = _vp()
    with _Temps() as t:
        _check(lib().gfq_rrf(t.bit(u), b.h, c.h, ctypes.byref(h)))
    return _mat(h)


def crz(m, lam, out_cols: int) -> Matrix:
    m = _as_matrix(m)
    h = _vp()
    with _Temps() as t:
        _check(lib().gfq_crz(m.h, t.bit(lam), out_cols, ctypes.byref(h)))
    return _mat(h)


def adi(k, delta) -> Matrix:
    k = _as_matrix(k)
    h = _vp()
    with _Temps() as t:
        _check(lib().gfq_adi(k.h, t.bit(delta), ctypes.byref(h)))
    return _mat(h)


# ---------------------------------------------------------------- packages / tasks
@dataclass
class PkgA:
    """reference include/gfrref/packages.hpp:17-26"""
    M: Matrix
    K: Matrix
    rho_prime: IndexSet
    A: Optional[Matrix] = None
    E: Optional[Matrix] = None
    lam: Optional[BitString] = None

    def _struct(self, t: _Temps):
        return _capi.PkgA(_opt_h(self.A), self.M.h, self.K.h, t.iset(self.rho_prime), _opt_h(self.E),
                          t.bit(self.lam) if self.lam is not None else None)

    @staticmethod
    def _take(s: _capi.PkgA) -> "PkgA":
        return PkgA(_mat(s.M), _mat(s.K), IndexSet._take(s.rho_prime), _mat(s.A) if s.A else None,
                    _mat(s.E) if s.E else None, BitString._take(s.lam) if s.lam else None)


@dataclass
class PkgD:
    """reference include/gfrref/packages.hpp:30-36"""
    R: Matrix = None
    gamma: IndexSet = field(default_factory=IndexSet)

    def rank(self):
        return len(self.gamma)

    def _struct(self, t: _Temps):
        R = self.R if self.R is not None else Matrix.zeros(0, 0)
        self._keep = R
        return _capi.PkgD(R.h, t.iset(self.gamma))

    @staticmethod
    def _take(s: _capi.PkgD) -> "PkgD":
        return PkgD(_mat(s.R), IndexSet._take(s.gamma))


@dataclass
class PkgE:
    """reference include/gfrref/packages.hpp:40-45"""
    rho: IndexSet
    delta: BitString

    def _struct(self, t: _Temps):
        return _capi.PkgE(t.iset(self.rho), t.bit(self.delta))

    @staticmethod
    def _take(s: _capi.PkgE) -> "PkgE":
        return PkgE(IndexSet._take(s.rho), BitString._take(s.delta))


def clear_down(f: FieldSpec, C, D: Optional[PkgD], i: int, ech_threshold: int = 256):
    """reference tasks.hpp:19 -> (PkgD, PkgA)"""
    C = _as_matrix(C, f)
    dout, aout = _capi.PkgD(), _capi.PkgA()
    with _Temps() as t:
        dp = ctypes.byref(D._struct(t)) if (D is not None and i > 0) else None
        if D is not None and i == 0:
            dp = None
        _check(lib().gfq_clear_down(f.code, C.h, dp, i, ech_threshold, ctypes.byref(dout), ctypes.byref(aout)))
    return PkgD._take(dout), PkgA._take(aout)


def update_row(f: FieldSpec, A: PkgA, C, B: Optional[Matrix], i: int):
    """reference tasks.hpp:26 -> (C', B')"""
    C = _as_matrix(C, f)
    B = _as_matrix(B, f) if B is not None else None
    co, bo = _vp(), _vp()
    with _Temps() as t:
        a = A._struct(t)
        _check(lib().gfq_update_row(f.code, ctypes.byref(a), C.h, _opt_h(B), i, ctypes.byref(co), ctypes.byref(bo)))
    return _mat(co), _mat(bo)


def update_row_trafo(f: FieldSpec, A: PkgA, K: Optional[Matrix], M: Optional[Matrix], E: PkgE, i: int,
                     h: int, j: int):
    """reference tasks.hpp:36 -> (K', M')"""
    K = _as_matrix(K, f) if K is not None else None
    M = _as_matrix(M, f) if M is not None else None
    ko, mo = _vp(), _vp()
    with _Temps() as t:
        a, e = A._struct(t), E._struct(t)
        _check(lib().gfq_update_row_trafo(f.code, ctypes.byref(a), _opt_h(K), _opt_h(M), ctypes.byref(e), i, h, j,
                                          ctypes.byref(ko), ctypes.byref(mo)))
    return _mat(ko), _mat(mo)


def extend(A: PkgA, E: Optional[PkgE], j: int) -> PkgE:
    """reference tasks.hpp:44"""
    out = _capi.PkgE()
    with _Temps() as t:
        a = A._struct(t)
        e = E._struct(t) if E is not None else None
        _check(lib().gfq_extend(ctypes.byref(a), ctypes.byref(e) if e is not None else None, j, ctypes.byref(out)))
    return PkgE._take(out)


def row_lengthen(M, E1: PkgE, E2: PkgE) -> Matrix:
    """reference tasks.hpp:48"""
    M = _as_matrix(M)
    h = _vp()
    with _Temps() as t:
        e1, e2 = E1._struct(t), E2._struct(t)
        _check(lib().gfq_row_lengthen(M.h, ctypes.byref(e1), ctypes.byref(e2), ctypes.byref(h)))
    return _mat(h)


def pre_clear_up(B, D: PkgD):
    """reference tasks.hpp:52 -> (X, R)"""
    B = _as_matrix(B)
    x, r = _vp(), _vp()
    with _Temps() as t:
        d = D._struct(t)
        _check(lib().gfq_pre_clear_up(B.h, ctypes.byref(d), ctypes.byref(x), ctypes.byref(r)))
    return _mat(x), _mat(r)


def clear_up(f: FieldSpec, R, X, M) -> Matrix:
    """reference tasks.hpp:55 (R + X.M)"""
    R, X, M = _as_matrix(R, f), _as_matrix(X, f), _as_matrix(M, f)
    h = _vp()
    _check(lib().gfq_clear_up(f.code, R.h, X.h, M.h, ctypes.byref(h)))
    return _mat(h)


def copy_d(D: PkgD) -> Matrix:
    """reference tasks.hpp:58"""
    h = _vp()
    with _Temps() as t:
        d = D._struct(t)
        _check(lib().gfq_copy_d(ctypes.byref(d), ctypes.byref(h)))
    return _mat(h)


# ---------------------------------------------------------------- chief
@dataclass
class ChopSpec:
    """reference include/gfrref/chief.hpp:15-25"""
    row_parts: list
    col_parts: list

    def a(self):
        return len(self.row_parts)

    def b(self):
        return len(self.col_parts)

    def rows(self):
        return sum(self.row_parts)

    def cols(self):
        return sum(self.col_parts)

    def row_offset(self, i):
        return sum(self.row_parts[:i])

    def col_offset(self, j):
        return sum(self.col_parts[:j])


def chop(m: int, n: int, block: int, remainder_first: bool = False) -> ChopSpec:
    """reference chief.hpp:27 (ChopMatrix)"""
    a, b = ctypes.c_uint64(), ctypes.c_uint64()
    _check(raw_lib().gfq_chop(m, n, block, int(remainder_first), None, ctypes.byref(a), None, ctypes.byref(b)))
    rp = (ctypes.c_uint64 * max(a.value, 1))()
    cp = (ctypes.c_uint64 * max(b.value, 1))()
    _check(raw_lib().gfq_chop(m, n, block, int(remainder_first), rp, None, cp, None))
    return ChopSpec([int(x) for x in rp[: a.value]], [int(x) for x in cp[: b.value]])


@dataclass
class EchelonizeOptions:
    """reference include/gfrref/chief.hpp:76-84 (`threads` = host workers,
    one CUDA stream each)."""
    block: int = 256
    threads: int = 1
    with_transform: bool = True
    ech_threshold: int = 256
    remainder_first: bool = False
    collect_trace: bool = False
    retain_all: bool = False
    fuse: bool = True  # wide UpdateRow / ClearUp jobs per panel (single GPU); False = reference task grid

    def _struct(self):
        return _capi.Options(self.block, self.threads, int(self.with_transform), self.ech_threshold,
                             int(self.remainder_first), int(self.collect_trace), int(self.retain_all),
                             int(self.fuse))


TASK_KINDS = ["ClearDown", "UpdateRow", "UpdateRowTrafo", "Extend", "RowLengthen", "PreClearUp", "ClearUp", "Copy",
              "UpdateRowW", "ClearUpRW", "ClearUpMW", "UpdateRowTrafoW"]


class EchelonOutput:
    """reference include/gfrref/chief.hpp:33-59 over a ``gfq_output`` handle."""

    def __init__(self, handle, field_: FieldSpec, chop_: ChopSpec, with_transform: bool):
        self.h = handle
        self.field = field_
        self.chop = chop_
        self.with_transform = with_transform
        r = ctypes.c_uint64()
        _check(lib().gfq_output_rank(handle, ctypes.byref(r)))
        self.rank = r.value
        a, b = chop_.a(), chop_.b()
        self.upsilon = [self._select(0, j, chop_.col_parts[j]) for j in range(b)]
        self.varrho = [self._select(1, i, chop_.row_parts[i]) for i in range(a)]
        self._cache = {}

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.gfq_output_free(self.h)
            self.h = None

    def _select(self, which, x, universe):
        n = ctypes.c_uint64()
        _check(lib().gfq_output_select(self.h, which, x, None, ctypes.byref(n)))
        buf = np.zeros(max(n.value, 1), np.uint32)
        _check(lib().gfq_output_select(self.h, which, x, buf.ctypes.data_as(_capi.c_u32p), None))
        return IndexSet(universe, tuple(buf[: n.value].tolist()))

    def block(self, kind: int, x: int, y: int) -> Matrix:
        key = (kind, x, y)
        if key not in self._cache:
            h = _vp()
            _check(lib().gfq_output_block(self.h, kind, x, y, ctypes.byref(h)))
            self._cache[key] = _mat(h)
        return self._cache[key]

    @property
    def R_blocks(self):
        b = self.chop.b()
        return [[self.block(0, j, l) if l >= j else None for l in range(b)] for j in range(b)]

    @property
    def T_M_blocks(self):
        if not self.with_transform:
            return []
        return [[self.block(1, j, h) for h in range(self.chop.a())] for j in range(self.chop.b())]

    @property
    def T_K_blocks(self):
        if not self.with_transform:
            return []
        return [[self.block(2, i, h) for h in range(i + 1)] for i in range(self.chop.a())]

    def global_upsilon(self):
        return [self.chop.col_offset(j) + v for j, s in enumerate(self.upsilon) for v in s.members]

    def global_varrho(self):
        return [self.chop.row_offset(i) + v for i, s in enumerate(self.varrho) for v in s.members]

    def assembled_R(self) -> Matrix:
        h = _vp()
        _check(lib().gfq_output_assembled_R(self.h, ctypes.byref(h)))
        return _mat(h)

    def materialize_transform(self) -> Matrix:
        h = _vp()
        _check(lib().gfq_output_transform(self.h, ctypes.byref(h)))
        return _mat(h)

    def block_bytes(self) -> int:
        n = ctypes.c_uint64()
        _check(lib().gfq_output_block_bytes(self.h, ctypes.byref(n)))
        return n.value

    def download_blocks(self, buf: np.ndarray) -> int:
        """D2H of every R / T_M / T_K block into `buf` (pinned or pageable)."""
        n = self.block_bytes()
        assert buf.nbytes >= n
        _check(lib().gfq_output_download_blocks(self.h, buf.ctypes.data_as(_capi.c_u8p), buf.nbytes))
        return n

    def write_selects_file(self, path: str):
        """reference write_selects_file (src/io.cpp:261), byte-identical."""
        _check(lib().gfq_output_write_selects_file(self.h, os.fsencode(path)))

    def write_transform_file(self, path: str):
        """reference write_transform_file (src/io.cpp:288), byte-identical."""
        _check(lib().gfq_output_write_transform_file(self.h, os.fsencode(path)))

    def report(self) -> dict:
        r = _capi.Report()
        _check(lib().gfq_output_report(self.h, ctypes.byref(r)))
        return dict(wall_ns=r.wall_ns, peak_live_bytes=r.peak_live_bytes,
                    initial_live_bytes=r.initial_live_bytes, tasks=r.tasks, workers=r.workers)

    def trace(self):
        n = ctypes.c_uint64()
        _check(lib().gfq_output_trace(self.h, ctypes.byref(n), *([None] * 8)))
        cnt = n.value
        arrs = [np.zeros(max(cnt, 1), np.int32) for _ in range(6)] + [np.zeros(max(cnt, 1), np.int64)
                                                                      for _ in range(2)]
        kind, i, j, k, w, det, s, e = arrs
        _check(lib().gfq_output_trace(self.h, None, *(a.ctypes.data_as(_capi.c_i32p) for a in (kind, i, j, k, w)),
                                      s.ctypes.data_as(_capi.c_i64p), e.ctypes.data_as(_capi.c_i64p),
                                      det.ctypes.data_as(_capi.c_i32p)))
        ds, de = np.zeros(max(cnt, 1), np.int64), np.zeros(max(cnt, 1), np.int64)
        _check(lib().gfq_output_trace_device(self.h, None, ds.ctypes.data_as(_capi.c_i64p),
                                             de.ctypes.data_as(_capi.c_i64p)))
        live = np.zeros(max(cnt, 1), np.int64)
        _check(lib().gfq_output_trace_live(self.h, None, live.ctypes.data_as(_capi.c_i64p)))
        return [dict(kind=TASK_KINDS[kind[q]], i=int(i[q]), j=int(j[q]), k=int(k[q]), worker=int(w[q]),
                     start_ns=int(s[q]), end_ns=int(e[q]), detail=int(det[q]),
                     dev_start_ns=int(ds[q]), dev_end_ns=int(de[q]), live_bytes=int(live[q]))
                for q in range(cnt)]


def echelonize(C, f: FieldSpec, options: EchelonizeOptions = None, host_out=None) -> EchelonOutput:
    """reference chief.hpp:88-90.  C: a device ``Matrix`` or a host uint8
    array (copied to HBM inside the call).  host_out (host C only): a uint8
    array of at least block_bytes() bytes receiving every output block in
    download_blocks' layout, each copied as soon as it is final."""
    options = options or EchelonizeOptions()
    o = options._struct()
    h = _vp()
    if f.wide and not isinstance(C, Matrix):
        if host_out is not None:
            raise ValueError("echelonize: host_out needs a u8 field")
        C = Matrix.from_numpy(C, 4)  # wide fields: u32 elements on the device
    if host_out is not None:
        if isinstance(C, Matrix):
            raise ValueError("echelonize: host_out needs a host input")
        a = np.ascontiguousarray(np.asarray(C, np.uint8))
        m, n = a.shape
        src = a if a.size else np.zeros(1, np.uint8)
        _check(lib().gfq_echelonize_host_into(f.code, m, n, src.ctypes.data_as(_capi.c_u8p), max(n, 1),
                                              ctypes.byref(o), host_out.ctypes.data_as(_capi.c_u8p),
                                              host_out.nbytes, ctypes.byref(h)))
        return EchelonOutput(h, f, chop(m, n, options.block, options.remainder_first), options.with_transform)
    if isinstance(C, Matrix):
        m, n = C.rows, C.cols
        _check(lib().gfq_echelonize(f.code, C.h, ctypes.byref(o), ctypes.byref(h)))
    else:
        a = np.ascontiguousarray(np.asarray(C, np.uint8))
        m, n = a.shape
        src = a if a.size else np.zeros(1, np.uint8)
        _check(lib().gfq_echelonize_host(f.code, m, n, src.ctypes.data_as(_capi.c_u8p), max(n, 1), ctypes.byref(o),
                                         ctypes.byref(h)))
    return EchelonOutput(h, f, chop(m, n, options.block, options.remainder_first), options.with_transform)


# ---------------------------------------------------------------- multi-GPU
class Comm:
    """Broadcast communicator of the sharded Chief (``gfq_comm``)."""

    def __init__(self, handle, rank, world):
        self.h, self.rank, self.world = handle, rank, world

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.gfq_comm_free(self.h)
            self.h = None

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (ctypes.c_uint8 * 128)()
        _check(lib().gfq_nccl_unique_id(buf))
        return bytes(buf)

    @staticmethod
    def nccl(world: int, rank: int, unique_id: bytes) -> "Comm":
        """One process per GPU; `unique_id` from rank 0's nccl_unique_id()."""
        h = _vp()
        idb = (ctypes.c_uint8 * 128)(*unique_id)
        _check(lib().gfq_comm_nccl(world, rank, idb, ctypes.byref(h)))
        return Comm(h, rank, world)

    @staticmethod
    def loopback(world: int):
        """`world` ranks in this process on the current GPU (each must be
        driven from its own thread)."""
        arr = (ctypes.c_void_p * world)()
        _check(lib().gfq_comm_loopback(world, arr))
        return [Comm(ctypes.c_void_p(arr[r]), r, world) for r in range(world)]


def echelonize_dist(comm: Comm, f: FieldSpec, m: int, n: int, options: EchelonizeOptions = None,
                    C: Matrix = None, seed: int = 0, gather: bool = True) -> EchelonOutput:
    """Sharded echelonize on this rank (block columns owned round-robin).
    C: full device input (only owned columns are read) or None to generate
    random_matrix(p, m, n, seed) columns on the device."""
    options = options or EchelonizeOptions()
    o = options._struct()
    h = _vp()
    _check(lib().gfq_echelonize_dist(comm.h, f.code, C.h if C is not None else None, m, n, seed,
                                     ctypes.byref(o), int(gather), ctypes.byref(h)))
    return EchelonOutput(h, f, chop(m, n, options.block, options.remainder_first), options.with_transform)


def read_gfmat_file(path: str):
    """reference read_gfmat_file (src/io.cpp:215): (FieldSpec, device Matrix)."""
    p = ctypes.c_uint32()
    h = _vp()
    _check(lib().gfq_read_gfmat_file(os.fsencode(path), ctypes.byref(p), ctypes.byref(h)))
    return FieldSpec.from_code(p.value), _mat(h)


def write_gfmat_file(path: str, f: FieldSpec, m) -> None:
    """reference write_gfmat_file (src/io.cpp:228), byte-identical."""
    m = _as_matrix(m, f)
    _check(lib().gfq_write_gfmat_file(os.fsencode(path), f.code, m.h))


VERIFY_METHODS = {"auto": 0, "exact": 1, "freivalds": 2}


def verify(C, out: EchelonOutput, method: str = "auto", seed: int = 1):
    """reference gfrref::verify (src/chief.cpp:531-590), on the device and
    without the oracle argument (gfq_verify).  Returns (ok, diag, checked):
    `checked` is "exact" (T materialised, T.C compared), "freivalds"
    (T.(C.X) vs E.X, X random n x 64) or "row-space" (no transform)."""
    C = _as_matrix(C, out.field)
    ok = ctypes.c_int32()
    diag = ctypes.create_string_buffer(512)
    chk = ctypes.create_string_buffer(32)
    _check(lib().gfq_verify(out.h, C.h, VERIFY_METHODS[method], seed, ctypes.byref(ok), diag, 512, chk, 32))
    return bool(ok.value), diag.value.decode(), chk.value.decode()


def dist_plan(m: int, n: int, block: int, with_transform: bool, world: int):
    """Host-only view of the sharded plan: ([(kind, i, j, k, owner)], [(is_a, i, j, k, root)])."""
    nn, nb = ctypes.c_uint64(), ctypes.c_uint64()
    L = raw_lib()
    _check(L.gfq_dist_plan(m, n, block, int(with_transform), world, None, ctypes.byref(nn), None,
                           ctypes.byref(nb)))
    nodes = np.zeros(5 * max(nn.value, 1), np.int32)
    bc = np.zeros(5 * max(nb.value, 1), np.int32)
    _check(L.gfq_dist_plan(m, n, block, int(with_transform), world, nodes.ctypes.data_as(_capi.c_i32p), None,
                           bc.ctypes.data_as(_capi.c_i32p), None))
    nodes = [(TASK_KINDS[r[0]], int(r[1]), int(r[2]), int(r[3]), int(r[4]))
             for r in nodes[: 5 * nn.value].reshape(-1, 5)]
    bcasts = [(bool(r[0]), int(r[1]), int(r[2]), int(r[3]), int(r[4])) for r in bc[: 5 * nb.value].reshape(-1, 5)]
    return nodes, bcasts


def random_matrix(f: FieldSpec, rows: int, cols: int, seed: int) -> Matrix:
    """reference generate.hpp:33-35, generated on the device (K6)."""
    h = _vp()
    _check(lib().gfq_random_matrix(f.code, rows, cols, seed, ctypes.byref(h)))
    return _mat(h)


def random_product_matrix(f: FieldSpec, rows: int, cols: int, inner: int, seed: int) -> Matrix:
    """reference generate.hpp:37-39 (K6 + K1)."""
    h = _vp()
    _check(lib().gfq_random_product_matrix(f.code, rows, cols, inner, seed, ctypes.byref(h)))
    return _mat(h)


def mad_raw(p: int, m: int, n: int, k: int, A: int, lda: int, B: int, ldb: int, Cin: int, ldc: int, D: int,
            ldd: int):
    """K1 on raw device pointers (ints), ordered on the current stream."""
    _check(lib().gfq_mad_raw(p, m, n, k, A, lda, B, ldb, Cin or None, ldc, D, ldd))


def set_mad_policy(policy: int):
    _check(lib().gfq_set_mad_policy(policy))


def mad_counters(reset: bool = False):
    s, t = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().gfq_mad_counters(ctypes.byref(s), ctypes.byref(t), int(reset)))
    return s.value, t.value


def set_ech_base(n: int):
    _check(lib().gfq_set_ech_base(n))


def set_ech_outer(width: int):
    """Outer panel width of the two-level device ECH (-1 auto, 0 one level)."""
    _check(lib().gfq_set_ech_outer(width))


def reserve_for(m: int, n: int, with_transform: bool = True):
    """Reserve the device pool for an m x n echelonize up front (gfq_reserve_for)."""
    _check(lib().gfq_reserve_for(m, n, int(with_transform)))


def set_poison(mode: int):
    """Developer check: bit 0 poisons allocations (0xA5), bit 1 freed blocks (0x5A)."""
    _check(lib().gfq_set_poison(mode))


def set_ech_mode(mode: int):
    """0 = device ECH (default: GF(2) blocks beyond the cluster kernel split by the
    reference rule), 1 = reference split/combine recursion over the small base
    kernel, 2 = device ECH with tall GF(2) blocks on the two-level path with
    single-CTA panel steps, 3 = as 0, 4 = device ECH with GF(2) blocks beyond the
    whole-block cluster kernel on the two-level path, one cluster launch per
    outer panel (ech_gf2_outer)."""
    _check(lib().gfq_set_ech_mode(mode))


def launch_count(reset: bool = False) -> int:
    v = ctypes.c_int64()
    _check(lib().gfq_launch_count(int(reset), ctypes.byref(v)))
    return v.value


def profile(on: bool):
    _check(lib().gfq_profile(int(on)))


def profile_take():
    """K1 per-launch device timing since the last take:
    {"tc": (launches, ops, ms), "simt": (launches, ops, ms)}."""
    l = (ctypes.c_int64 * 2)()
    o = (ctypes.c_double * 2)()
    t = (ctypes.c_double * 2)()
    _check(lib().gfq_profile_take(l, o, t))
    return {"tc": (l[0], o[0], t[0]), "simt": (l[1], o[1], t[1])}


def device_memory(reset_peak: bool = False) -> dict:
    """The library's device bytes: live, high-water since the last reset,
    and the stream-ordered pool's reserved high-water."""
    live, peak, res = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _check(lib().gfq_device_memory(int(reset_peak), ctypes.byref(live), ctypes.byref(peak), ctypes.byref(res)))
    return {"live": live.value, "peak": peak.value, "pool_reserved_high": res.value}


PROFILE_KINDS = ("k1_tc", "k1_simt", "ech_gf2", "ech_panel", "select", "k1_f4")


def profile_take_kinds(with_union: bool = False):
    """Per kernel family since the last take: {name: (launches, work, ms)}
    (+ union_ms, the time any launch of the family ran, with_union);
    work = int8 ops for k1_*, algorithmic bytes for the others."""
    n = len(PROFILE_KINDS)
    l = (ctypes.c_int64 * n)()
    w = (ctypes.c_double * n)()
    t = (ctypes.c_double * n)()
    u = (ctypes.c_double * n)()
    _check(lib().gfq_profile_take_kinds(n, l, w, t, u))
    if with_union:
        return {name: (l[q], w[q], t[q], u[q]) for q, name in enumerate(PROFILE_KINDS)}
    return {name: (l[q], w[q], t[q]) for q, name in enumerate(PROFILE_KINDS)}


def set_host_pack(on):
    """GF(2) host buffers cross PCIe packed 8:1 (off by default).  An int
    N >= 2 selects the hybrid: every N-th block row / output block packed,
    the rest as byte copies (host packing and PCIe run side by side)."""
    _check(lib().gfq_set_host_pack(int(on)))


def last_transfer_bytes():
    """(h2d, d2h): bytes that crossed PCIe in this thread's last host-buffer
    echelonize (GF(2) buffers travel packed 8:1)."""
    h, d = ctypes.c_int64(0), ctypes.c_int64(0)
    _check(lib().gfq_last_transfer_bytes(ctypes.byref(h), ctypes.byref(d)))
    return h.value, d.value


def set_stream(stream_ptr: int):
    _check(lib().gfq_set_stream(stream_ptr or None))


def synchronize():
    _check(lib().gfq_synchronize())
