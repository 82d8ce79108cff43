"""TEST INFRASTRUCTURE ONLY -- the CPU checker for the B200 GF(p) RREF path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product (``paper_1806_04211_b200``) never imports it; its compute path is the
CUDA library and fails loudly when that is missing.

Contents
--------
``lib``      ctypes handle on ``oracle/liboracle.so`` -- the plain-C restatement
             (``gfq_oracle.c``) of the reference's generators, block
             multiply-accumulate and sequential RREF oracle.
``ref``      ctypes handle on ``oracle/_ref/libgfrref_ref.so`` -- the reference
             library itself, compiled from /root/reference by ``oracle/Makefile``
             (None when that build is absent).
``restate``  numpy restatement of the reference's jobs, tasks and Chief plan
             (``restate.py``), used as the task-level checker.

Parity pin: ``tests/test_oracle.py`` checks all three against the golden
vectors in ``tests/golden/`` (values from the reference's own test suite) and
against each other.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(HERE, "liboracle.so")
_REF_PATH = os.path.join(HERE, "_ref", "libgfrref_ref.so")

_u8p = ctypes.POINTER(ctypes.c_uint8)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_sz = ctypes.c_size_t


def _build_if_missing():
    if not os.path.exists(_LIB_PATH):
        subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)


def _load():
    _build_if_missing()
    lib = ctypes.CDLL(_LIB_PATH)
    lib.gfo_random_matrix.argtypes = [ctypes.c_uint32, _sz, _sz, ctypes.c_uint64, _u8p, _sz]
    lib.gfo_random_product_matrix.argtypes = [ctypes.c_uint32, _sz, _sz, _sz, ctypes.c_uint64, _u8p, _sz]
    lib.gfo_mad.argtypes = [ctypes.c_uint32, _sz, _sz, _sz, _u8p, _sz, _u8p, _sz, _u8p, _sz, _u8p, _sz]
    lib.gfo_oracle_rref.argtypes = [ctypes.c_uint32, _sz, _sz, _u8p, _sz, _u32p, _u32p, _u8p, _u8p, _u8p]
    lib.gfo_oracle_rref.restype = ctypes.c_int64
    lib.gfo_inv.argtypes = [ctypes.c_uint32, ctypes.c_uint32]
    lib.gfo_inv.restype = ctypes.c_uint32
    lib.gfo_field_ext.argtypes = [ctypes.c_uint32, ctypes.c_uint32, _u32p]
    lib.gfo_field_ext.restype = ctypes.c_uint32
    for fn in (lib.gfo_add, lib.gfo_mul):
        fn.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32]
        fn.restype = ctypes.c_uint32
    lib.gfo_neg.argtypes = [ctypes.c_uint32, ctypes.c_uint32]
    lib.gfo_neg.restype = ctypes.c_uint32
    lib.gfo_order.argtypes = [ctypes.c_uint32]
    lib.gfo_order.restype = ctypes.c_uint32
    return lib


def _load_ref():
    if not os.path.exists(_REF_PATH):
        return None
    r = ctypes.CDLL(_REF_PATH)
    r.ref_last_error.restype = ctypes.c_char_p
    r.ref_hardware_concurrency.restype = ctypes.c_int
    r.ref_random_matrix.argtypes = [ctypes.c_uint32, _sz, _sz, ctypes.c_uint64, _u8p, _sz]
    r.ref_random_product_matrix.argtypes = [ctypes.c_uint32, _sz, _sz, _sz, ctypes.c_uint64, _u8p, _sz]
    r.ref_mad.argtypes = [ctypes.c_uint32, _sz, _sz, _sz, _u8p, _sz, _u8p, _sz, _u8p, _sz, _u8p, _sz]
    r.ref_mad.restype = ctypes.c_int
    for fn in (r.ref_ech, r.ref_oracle_rref):
        fn.restype = ctypes.c_int64
    r.ref_ech.argtypes = [ctypes.c_uint32, _sz, _sz, _u8p, _sz, _sz, _u32p, _u32p, _u8p, _u8p, _u8p]
    r.ref_oracle_rref.argtypes = [ctypes.c_uint32, _sz, _sz, _u8p, _sz, _u32p, _u32p, _u8p, _u8p, _u8p]
    r.ref_echelonize.restype = ctypes.c_void_p
    r.ref_echelonize.argtypes = [ctypes.c_uint32, _sz, _sz, _u8p, _sz, _sz, ctypes.c_int, ctypes.c_int, _sz,
                                 ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
    r.ref_out_free.argtypes = [ctypes.c_void_p]
    for fn in (r.ref_out_rank, r.ref_out_a, r.ref_out_b):
        fn.restype = ctypes.c_int64
        fn.argtypes = [ctypes.c_void_p]
    r.ref_out_select.restype = ctypes.c_int64
    r.ref_out_select.argtypes = [ctypes.c_void_p, ctypes.c_int, _sz, _u32p]
    r.ref_out_block.restype = ctypes.c_int
    r.ref_out_block.argtypes = [ctypes.c_void_p, ctypes.c_int, _sz, _sz, ctypes.POINTER(ctypes.c_int64),
                                ctypes.POINTER(ctypes.c_int64), _u8p]
    r.ref_out_materialize.argtypes = [ctypes.c_void_p, _u8p]
    r.ref_out_assembled_R.argtypes = [ctypes.c_void_p, _u8p]
    r.ref_verify.argtypes = [ctypes.c_void_p, ctypes.c_uint32, _sz, _sz, _u8p, _sz]
    r.ref_field_register.argtypes = [ctypes.c_uint32, ctypes.c_uint32, _u32p, _sz]
    r.ref_field_register.restype = ctypes.c_uint32
    r.ref_field_op.argtypes = [ctypes.c_uint32, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32]
    r.ref_field_op.restype = ctypes.c_uint32
    r.ref_default_modulus.argtypes = [ctypes.c_uint32, ctypes.c_uint32, _u32p]
    r.ref_set_elem_bytes.argtypes = [ctypes.c_int]
    return r


def _need_ref():
    if ref is None:
        raise RuntimeError("reference library oracle/_ref/libgfrref_ref.so not built")
    return ref


lib = _load()
ref = _load_ref()


def u8ptr(a: np.ndarray):
    if a is None:
        return None
    assert a.dtype == np.uint8 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_u8p)


def u32ptr(a: np.ndarray):
    assert a.dtype == np.uint32 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_u32p)


def ext_code(p: int, k: int, modulus) -> int:
    """Code of GF(p^k) with this modulus in the C restatement (q <= 256);
    every oracle function takes it in place of p."""
    m = np.ascontiguousarray(np.asarray(modulus, np.uint32))
    code = lib.gfo_field_ext(p, k, u32ptr(m))
    if code == 0:
        raise ValueError(f"oracle: cannot build GF({p}^{k}) with modulus {list(modulus)}")
    return int(code)


def field_op(code: int, op: str, a: int, b: int = 0) -> int:
    if op == "add":
        return int(lib.gfo_add(code, a, b))
    if op == "mul":
        return int(lib.gfo_mul(code, a, b))
    if op == "neg":
        return int(lib.gfo_neg(code, a))
    return int(lib.gfo_inv(code, a))


def ref_ext_code(p: int, k: int, modulus=None) -> int:
    """Code of the reference library's FieldSpec(p, k, modulus) for the ref_*
    functions (oracle/ref_shim.cpp)."""
    r = _need_ref()
    if modulus is None:
        code = r.ref_field_register(p, k, None, 0)
    else:
        m = np.ascontiguousarray(np.asarray(modulus, np.uint32))
        code = r.ref_field_register(p, k, u32ptr(m), m.size)
    if code == 0:
        raise ValueError(r.ref_last_error().decode())
    return int(code)


def ref_field_op(code: int, op: str, a: int, b: int = 0) -> int:
    return int(_need_ref().ref_field_op(code, {"add": 0, "mul": 1, "neg": 2, "inv": 3}[op], a, b))


def ref_default_modulus(p: int, k: int):
    out = np.zeros(k + 1, np.uint32)
    _need_ref().ref_default_modulus(p, k, u32ptr(out))
    return [int(x) for x in out]


def random_matrix(p: int, rows: int, cols: int, seed: int) -> np.ndarray:
    """C restatement of reference ``random_matrix`` (src/generate.cpp:16-24)."""
    out = np.zeros((rows, cols), np.uint8)
    lib.gfo_random_matrix(p, rows, cols, seed, u8ptr(out), max(cols, 1))
    return out


def random_product_matrix(p: int, rows: int, cols: int, inner: int, seed: int) -> np.ndarray:
    """C restatement of reference ``random_product_matrix`` (src/generate.cpp:26-38)."""
    out = np.zeros((rows, cols), np.uint8)
    lib.gfo_random_product_matrix(p, rows, cols, inner, seed, u8ptr(out), max(cols, 1))
    return out


def mad(p: int, a: np.ndarray, b: np.ndarray, c: np.ndarray | None = None) -> np.ndarray:
    """C restatement of reference ``mul_add_kernel`` (src/matrix.cpp:81-133)."""
    a = np.ascontiguousarray(a, np.uint8)
    b = np.ascontiguousarray(b, np.uint8)
    m, k = a.shape
    k2, n = b.shape
    if k != k2:
        raise ValueError("mul: inner dimensions disagree")
    if c is not None:
        c = np.ascontiguousarray(c, np.uint8)
        if c.shape != (m, n):
            raise ValueError("mad: addend shape mismatch")
    out = np.zeros((m, n), np.uint8)
    if m and n:
        lib.gfo_mad(p, m, k, n, u8ptr(a) if a.size else u8ptr(np.zeros(1, np.uint8)), max(k, 1),
                    u8ptr(b) if b.size else u8ptr(np.zeros(1, np.uint8)), max(n, 1),
                    u8ptr(c) if c is not None else None, n, u8ptr(out), n)
    return out


def ref_mad(p: int, a: np.ndarray, b: np.ndarray, c: np.ndarray | None = None) -> np.ndarray:
    """The reference's own ``mat_mul`` / ``mat_mul_add`` (src/matrix.cpp:137-144)."""
    r = _need_ref()
    a = np.ascontiguousarray(a, np.uint8)
    b = np.ascontiguousarray(b, np.uint8)
    m, k = a.shape
    n = b.shape[1]
    out = np.zeros((m, n), np.uint8)
    z = np.zeros(1, np.uint8)
    if c is not None:
        c = np.ascontiguousarray(c, np.uint8)
    rc = r.ref_mad(p, m, k, n, u8ptr(a) if a.size else u8ptr(z), max(k, 1), u8ptr(b) if b.size else u8ptr(z),
                   max(n, 1), u8ptr(c) if c is not None else None, max(n, 1), u8ptr(out) if out.size else u8ptr(z),
                   max(n, 1))
    if rc != 0:
        raise RuntimeError(r.ref_last_error().decode())
    return out


REF_ECH = os.path.join(HERE, "_ref", "ref_ech")


def ref_cli(*args):
    """Run the reference-library driver oracle/_ref/ref_ech (reference
    read_gfmat / echelonize / write_* in its own process; see
    ref_ech_main.cpp).  Returns (exit code, stdout)."""
    r = subprocess.run([REF_ECH, *map(str, args)], capture_output=True, text=True)
    return r.returncode, r.stdout


def ref_write_gfmat(p: int, C: np.ndarray, path: str):
    """The reference's write_gfmat_file (src/io.cpp:228) on a host matrix."""
    C = np.ascontiguousarray(C, np.uint8)
    raw = path + ".raw"
    C.tofile(raw)
    rc, _ = ref_cli("gfmat", p, C.shape[0], C.shape[1], raw, path)
    os.remove(raw)
    if rc:
        raise RuntimeError("ref_ech gfmat failed")


def oracle_rref(p: int, C: np.ndarray):
    """C restatement of reference ``oracle_rref`` (src/chief.cpp:427-487).

    Returns dict(rank, rho, gamma, M, K, R) with the reference's conventions.
    """
    C = np.ascontiguousarray(C, np.uint8)
    m, n = C.shape
    rho = np.zeros(max(m, 1), np.uint32)
    gamma = np.zeros(max(n, 1), np.uint32)
    M = np.zeros(max(m * m, 1), np.uint8)
    K = np.zeros(max(m * m, 1), np.uint8)
    R = np.zeros(max(m * n, 1), np.uint8)
    src = C if C.size else np.zeros((1, 1), np.uint8)
    r = lib.gfo_oracle_rref(p, m, n, u8ptr(src), max(n, 1), u32ptr(rho), u32ptr(gamma),
                            u8ptr(M), u8ptr(K), u8ptr(R))
    if r < 0:
        raise MemoryError("oracle_rref: allocation failed")
    return dict(rank=int(r), rho=rho[:r].copy(), gamma=gamma[:r].copy(),
                M=M[: r * r].reshape(r, r).copy(), K=K[: (m - r) * r].reshape(m - r, r).copy(),
                R=R[: r * (n - r)].reshape(r, n - r).copy())


# ---------------------------------------------------------------- reference shim
class RefOutput:
    """Handle on a ``gfrref::EchelonOutput`` produced by the reference library."""


    def __init__(self, handle, m, n, wall_s, run_s):
        self.h = handle
        self.m, self.n = m, n
        self.wall_s, self.run_s = wall_s, run_s

    def __del__(self):
        if getattr(self, "h", None) and ref is not None:
            ref.ref_out_free(self.h)
            self.h = None

    @property
    def rank(self):
        return int(ref.ref_out_rank(self.h))

    @property
    def a(self):
        return int(ref.ref_out_a(self.h))

    @property
    def b(self):
        return int(ref.ref_out_b(self.h))

    def select(self, which: int, x: int) -> np.ndarray:
        cnt = ref.ref_out_select(self.h, which, x, None)
        buf = np.zeros(max(cnt, 1), np.uint32)
        ref.ref_out_select(self.h, which, x, u32ptr(buf))
        return buf[:cnt].copy()

    def upsilon(self, j):
        return self.select(0, j)

    def varrho(self, i):
        return self.select(1, i)

    def block(self, kind: int, x: int, y: int) -> np.ndarray:
        rows, cols = ctypes.c_int64(), ctypes.c_int64()
        if ref.ref_out_block(self.h, kind, x, y, ctypes.byref(rows), ctypes.byref(cols), None):
            raise IndexError(ref.ref_last_error().decode())
        buf = np.zeros((rows.value, cols.value), np.uint8)
        if buf.size:
            ref.ref_out_block(self.h, kind, x, y, ctypes.byref(rows), ctypes.byref(cols), u8ptr(buf))
        return buf

    def materialize_transform(self) -> np.ndarray:
        t = np.zeros((self.m, self.m), np.uint8)
        if t.size and ref.ref_out_materialize(self.h, u8ptr(t)):
            raise RuntimeError(ref.ref_last_error().decode())
        return t

    def assembled_R(self) -> np.ndarray:
        r = self.rank
        out = np.zeros((r, self.n - r), np.uint8)
        if out.size:
            ref.ref_out_assembled_R(self.h, u8ptr(out))
        return out


def ref_echelonize(p: int, C: np.ndarray, block: int, threads: int = 1, with_transform: bool = True,
                   threshold: int = 256) -> RefOutput:
    """Run the reference's own ``gfrref::echelonize`` (src/chief.cpp:322-386)."""
    if ref is None:
        raise RuntimeError("reference library oracle/_ref/libgfrref_ref.so not built")
    C = np.ascontiguousarray(C, np.uint8)
    m, n = C.shape
    wall, run = ctypes.c_double(), ctypes.c_double()
    src = C if C.size else np.zeros((1, 1), np.uint8)
    h = ref.ref_echelonize(p, m, n, u8ptr(src), max(n, 1), block, threads, int(with_transform), threshold,
                           ctypes.byref(wall), ctypes.byref(run))
    if not h:
        raise RuntimeError(ref.ref_last_error().decode())
    return RefOutput(h, m, n, wall.value, run.value)


def ref_ech(p: int, H: np.ndarray, threshold: int = 256):
    """The reference's own single-block ``ech`` (src/jobs.cpp:202-225)."""
    H = np.ascontiguousarray(H, np.uint8)
    m, n = H.shape
    rho = np.zeros(max(m, 1), np.uint32)
    gamma = np.zeros(max(n, 1), np.uint32)
    M = np.zeros(max(m * m, 1), np.uint8)
    K = np.zeros(max(m * m, 1), np.uint8)
    R = np.zeros(max(m * n, 1), np.uint8)
    src = H if H.size else np.zeros((1, 1), np.uint8)
    r = ref.ref_ech(p, m, n, u8ptr(src), max(n, 1), threshold, u32ptr(rho), u32ptr(gamma), u8ptr(M),
                    u8ptr(K), u8ptr(R))
    if r < 0:
        raise RuntimeError(ref.ref_last_error().decode())
    return dict(rank=int(r), rho=rho[:r].copy(), gamma=gamma[:r].copy(),
                M=M[: r * r].reshape(r, r).copy(), K=K[: (m - r) * r].reshape(m - r, r).copy(),
                R=R[: r * (n - r)].reshape(r, n - r).copy())


def ref_random_matrix(p: int, rows: int, cols: int, seed: int) -> np.ndarray:
    out = np.zeros((rows, cols), np.uint8)
    if out.size:
        ref.ref_random_matrix(p, rows, cols, seed, u8ptr(out), cols)
    return out


def ref_random_product_matrix(p: int, rows: int, cols: int, inner: int, seed: int) -> np.ndarray:
    out = np.zeros((rows, cols), np.uint8)
    if out.size:
        ref.ref_random_product_matrix(p, rows, cols, inner, seed, u8ptr(out), cols)
    return out


# ---------------------------------------------------------------- wide fields (u32 buffers)
# Fields whose elements do not fit a byte (GF(p), p > 251; GF(p^k),
# p^k > 256) cross the shim as u32 buffers: ref_set_elem_bytes(4) around
# each call (oracle/ref_shim.cpp).  TEST INFRASTRUCTURE ONLY.
class _Wide:
    def __enter__(self):
        _need_ref().ref_set_elem_bytes(4)

    def __exit__(self, *exc):
        ref.ref_set_elem_bytes(1)


def _raw(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_u8p)


def ref32_random_matrix(code: int, rows: int, cols: int, seed: int) -> np.ndarray:
    """The reference's random_matrix (src/generate.cpp:16-24) as u32."""
    out = np.zeros((rows, cols), np.uint32)
    if out.size:
        with _Wide():
            ref.ref_random_matrix(code, rows, cols, seed, _raw(out), cols)
    return out


def ref32_mad(code: int, a: np.ndarray, b: np.ndarray, c: np.ndarray | None = None) -> np.ndarray:
    """The reference's mat_mul / mat_mul_add (src/matrix.cpp:137-144) on u32 matrices."""
    a = np.ascontiguousarray(a, np.uint32)
    b = np.ascontiguousarray(b, np.uint32)
    m, k = a.shape
    n = b.shape[1]
    out = np.zeros((m, n), np.uint32)
    z = np.zeros(1, np.uint32)
    if c is not None:
        c = np.ascontiguousarray(c, np.uint32)
    with _Wide():
        rc = ref.ref_mad(code, m, k, n, _raw(a) if a.size else _raw(z), max(k, 1), _raw(b) if b.size else _raw(z),
                         max(n, 1), _raw(c) if c is not None else None, max(n, 1), _raw(out) if out.size else _raw(z),
                         max(n, 1))
    if rc != 0:
        raise RuntimeError(ref.ref_last_error().decode())
    return out


def ref32_ech(code: int, H: np.ndarray, threshold: int = 256):
    """The reference's single-block ech (src/jobs.cpp:202-225) on a u32 matrix."""
    H = np.ascontiguousarray(H, np.uint32)
    m, n = H.shape
    rho = np.zeros(max(m, 1), np.uint32)
    gamma = np.zeros(max(n, 1), np.uint32)
    M = np.zeros(max(m * m, 1), np.uint32)
    K = np.zeros(max(m * m, 1), np.uint32)
    R = np.zeros(max(m * n, 1), np.uint32)
    src = H if H.size else np.zeros((1, 1), np.uint32)
    with _Wide():
        r = ref.ref_ech(code, m, n, _raw(src), max(n, 1), threshold, u32ptr(rho), u32ptr(gamma), _raw(M), _raw(K),
                        _raw(R))
    if r < 0:
        raise RuntimeError(ref.ref_last_error().decode())
    return dict(rank=int(r), rho=rho[:r].copy(), gamma=gamma[:r].copy(),
                M=M[: r * r].reshape(r, r).copy(), K=K[: (m - r) * r].reshape(m - r, r).copy(),
                R=R[: r * (n - r)].reshape(r, n - r).copy())


class RefOutput32(RefOutput):
    """RefOutput whose blocks are u32 (wide fields)."""

    def block(self, kind: int, x: int, y: int) -> np.ndarray:
        rows, cols = ctypes.c_int64(), ctypes.c_int64()
        if ref.ref_out_block(self.h, kind, x, y, ctypes.byref(rows), ctypes.byref(cols), None):
            raise IndexError(ref.ref_last_error().decode())
        buf = np.zeros((rows.value, cols.value), np.uint32)
        if buf.size:
            with _Wide():
                ref.ref_out_block(self.h, kind, x, y, ctypes.byref(rows), ctypes.byref(cols), _raw(buf))
        return buf

    def materialize_transform(self) -> np.ndarray:
        t = np.zeros((self.m, self.m), np.uint32)
        if t.size:
            with _Wide():
                bad = ref.ref_out_materialize(self.h, _raw(t))
            if bad:
                raise RuntimeError(ref.ref_last_error().decode())
        return t

    def assembled_R(self) -> np.ndarray:
        r = self.rank
        out = np.zeros((r, self.n - r), np.uint32)
        if out.size:
            with _Wide():
                ref.ref_out_assembled_R(self.h, _raw(out))
        return out


def ref32_echelonize(code: int, C: np.ndarray, block: int, threads: int = 1, with_transform: bool = True,
                     threshold: int = 256) -> RefOutput32:
    """The reference's own gfrref::echelonize (src/chief.cpp:322-386) on a u32 matrix."""
    r = _need_ref()
    C = np.ascontiguousarray(C, np.uint32)
    m, n = C.shape
    wall, run = ctypes.c_double(), ctypes.c_double()
    src = C if C.size else np.zeros((1, 1), np.uint32)
    with _Wide():
        h = r.ref_echelonize(code, m, n, _raw(src), max(n, 1), block, threads, int(with_transform), threshold,
                             ctypes.byref(wall), ctypes.byref(run))
    if not h:
        raise RuntimeError(r.ref_last_error().decode())
    return RefOutput32(h, m, n, wall.value, run.value)
