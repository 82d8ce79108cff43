"""ctypes prototypes for the C ABI in include/gfq.h (libgfq.so).

The library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_1806_04211_b200/csrc``).  Loading fails loudly when it is
missing: there is no CPU fallback for any compute entry point.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GFQ_LIB_PATH") or os.path.join(HERE, "lib", "libgfq.so")  # override: A/B builds
HEADER = os.path.join(os.path.dirname(HERE), "include", "gfq.h")

c_u8p = ctypes.POINTER(ctypes.c_uint8)
c_u32p = ctypes.POINTER(ctypes.c_uint32)
c_i32p = ctypes.POINTER(ctypes.c_int32)
c_i64p = ctypes.POINTER(ctypes.c_int64)
c_u64p = ctypes.POINTER(ctypes.c_uint64)
vp = ctypes.c_void_p
vpp = ctypes.POINTER(ctypes.c_void_p)


class PkgA(ctypes.Structure):
    _fields_ = [("A", vp), ("M", vp), ("K", vp), ("rho_prime", vp), ("E", vp), ("lam", vp)]


class PkgD(ctypes.Structure):
    _fields_ = [("R", vp), ("gamma", vp)]


class PkgE(ctypes.Structure):
    _fields_ = [("rho", vp), ("delta", vp)]


class Options(ctypes.Structure):
    _fields_ = [("block", ctypes.c_uint64), ("threads", ctypes.c_int), ("with_transform", ctypes.c_int),
                ("ech_threshold", ctypes.c_uint64), ("remainder_first", ctypes.c_int),
                ("collect_trace", ctypes.c_int), ("retain_all", ctypes.c_int), ("fuse", ctypes.c_int)]


class Report(ctypes.Structure):
    _fields_ = [("wall_ns", ctypes.c_int64), ("peak_live_bytes", ctypes.c_int64),
                ("initial_live_bytes", ctypes.c_int64), ("tasks", ctypes.c_int64), ("workers", ctypes.c_int)]


I, U32, U64, I64 = ctypes.c_int, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int64
_P = ctypes.POINTER

PROTOS = {
    "gfq_last_error": (ctypes.c_char_p, []),
    "gfq_version": (I, []),
    "gfq_init": (I, [I]),
    "gfq_set_stream": (I, [vp]),
    "gfq_synchronize": (I, []),
    "gfq_mat_upload": (I, [I64, I64, c_u8p, I64, vpp]),
    "gfq_mat_upload32": (I, [I64, I64, c_u32p, I64, vpp]),
    "gfq_mat_esize": (I, [vp, ctypes.POINTER(ctypes.c_int)]),
    "gfq_last_transfer_bytes": (I, [ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]),
    "gfq_set_host_pack": (I, [ctypes.c_int]),
    "gfq_mat_copy_device": (I, [I64, I64, vp, I64, vpp]),
    "gfq_mat_shape": (I, [vp, c_i64p, c_i64p]),
    "gfq_mat_download": (I, [vp, c_u8p, I64]),
    "gfq_mat_device_ptr": (I, [vp, _P(vp), c_i64p]),
    "gfq_mat_free": (None, [vp]),
    "gfq_iset_create": (I, [U64, c_u32p, U64, vpp]),
    "gfq_iset_get": (I, [vp, c_u64p, c_u64p, c_u32p]),
    "gfq_iset_free": (None, [vp]),
    "gfq_bits_create": (I, [c_u8p, U64, vpp]),
    "gfq_bits_get": (I, [vp, c_u64p, c_u8p]),
    "gfq_bits_free": (None, [vp]),
    "gfq_mad_raw": (I, [U32, I64, I64, I64, vp, I64, vp, I64, vp, I64, vp, I64]),
    "gfq_set_mad_policy": (I, [I]),
    "gfq_mad_counters": (I, [c_i64p, c_i64p, I]),
    "gfq_random_matrix": (I, [U32, I64, I64, U64, vpp]),
    "gfq_random_product_matrix": (I, [U32, I64, I64, I64, U64, vpp]),
    "gfq_set_ech_base": (I, [U64]),
    "gfq_set_ech_outer": (I, [ctypes.c_int]),
    "gfq_field_register": (I, [U32, U32, ctypes.c_void_p, I, ctypes.c_void_p]),
    "gfq_field_info": (I, [U32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "gfq_field_op": (I, [U32, I, U32, U32, ctypes.c_void_p]),
    "gfq_default_modulus": (I, [U32, U32, ctypes.c_void_p]),
    "gfq_set_ech_mode": (I, [I]),
    "gfq_set_poison": (I, [I]),
    "gfq_reserve_for": (I, [I64, I64, I]),
    "gfq_launch_count": (I, [I, c_i64p]),
    "gfq_profile": (I, [I]),
    "gfq_device_memory": (I, [I, c_i64p, c_i64p, c_i64p]),
    "gfq_output_trace_live": (I, [vp, c_u64p, c_i64p]),
    "gfq_profile_take_kinds": (I, [I, c_i64p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                   ctypes.POINTER(ctypes.c_double)]),
    "gfq_profile_take": (I, [c_i64p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
    "gfq_mul": (I, [U32, vp, vp, vpp]),
    "gfq_mad": (I, [U32, vp, vp, vp, vpp]),
    "gfq_ech": (I, [U32, vp, U64, vpp, vpp, vpp, vpp, vpp]),
    "gfq_cex": (I, [vp, vp, vpp, vpp]),
    "gfq_rex": (I, [vp, vp, vpp, vpp]),
    "gfq_unh": (I, [vp, vp, vpp, vpp]),
    "gfq_un0": (I, [vp, vpp, vpp]),
    "gfq_mkr": (I, [vp, vp, vpp]),
    "gfq_rrf": (I, [vp, vp, vp, vpp]),
    "gfq_crz": (I, [vp, vp, U64, vpp]),
    "gfq_adi": (I, [vp, vp, vpp]),
    "gfq_clear_down": (I, [U32, vp, _P(PkgD), U64, U64, _P(PkgD), _P(PkgA)]),
    "gfq_update_row": (I, [U32, _P(PkgA), vp, vp, U64, vpp, vpp]),
    "gfq_update_row_trafo": (I, [U32, _P(PkgA), vp, vp, _P(PkgE), U64, U64, U64, vpp, vpp]),
    "gfq_extend": (I, [_P(PkgA), _P(PkgE), U64, _P(PkgE)]),
    "gfq_row_lengthen": (I, [vp, _P(PkgE), _P(PkgE), vpp]),
    "gfq_pre_clear_up": (I, [vp, _P(PkgD), vpp, vpp]),
    "gfq_clear_up": (I, [U32, vp, vp, vp, vpp]),
    "gfq_copy_d": (I, [_P(PkgD), vpp]),
    "gfq_pkgA_free": (None, [_P(PkgA)]),
    "gfq_pkgD_free": (None, [_P(PkgD)]),
    "gfq_pkgE_free": (None, [_P(PkgE)]),
    "gfq_chop": (I, [U64, U64, U64, I, c_u64p, c_u64p, c_u64p, c_u64p]),
    "gfq_options_default": (None, [_P(Options)]),
    "gfq_echelonize": (I, [U32, vp, _P(Options), vpp]),
    "gfq_echelonize_host": (I, [U32, I64, I64, c_u8p, I64, _P(Options), vpp]),
    "gfq_echelonize_host_into": (I, [U32, I64, I64, c_u8p, I64, _P(Options), c_u8p, U64, vpp]),
    "gfq_output_rank": (I, [vp, c_u64p]),
    "gfq_output_grid": (I, [vp, c_u64p, c_u64p]),
    "gfq_output_select": (I, [vp, I, U64, c_u32p, c_u64p]),
    "gfq_output_block": (I, [vp, I, U64, U64, vpp]),
    "gfq_output_assembled_R": (I, [vp, vpp]),
    "gfq_output_transform": (I, [vp, vpp]),
    "gfq_output_block_bytes": (I, [vp, c_u64p]),
    "gfq_output_download_blocks": (I, [vp, c_u8p, U64]),
    "gfq_output_report": (I, [vp, _P(Report)]),
    "gfq_output_trace": (I, [vp, c_u64p, c_i32p, c_i32p, c_i32p, c_i32p, c_i32p, c_i64p, c_i64p, c_i32p]),
    "gfq_output_trace_device": (I, [vp, c_u64p, c_i64p, c_i64p]),
    "gfq_output_free": (None, [vp]),
    "gfq_tc_debug_take": (I, [c_u64p]),
    "gfq_read_gfmat_file": (I, [ctypes.c_char_p, _P(U32), vpp]),
    "gfq_write_gfmat_file": (I, [ctypes.c_char_p, U32, vp]),
    "gfq_output_write_selects_file": (I, [vp, ctypes.c_char_p]),
    "gfq_output_write_transform_file": (I, [vp, ctypes.c_char_p]),
    "gfq_verify": (I, [vp, vp, I, U64, c_i32p, ctypes.c_char_p, ctypes.c_size_t, ctypes.c_char_p,
                       ctypes.c_size_t]),
    "gfq_nccl_unique_id": (I, [c_u8p]),
    "gfq_comm_nccl": (I, [I, I, c_u8p, vpp]),
    "gfq_comm_loopback": (I, [I, vpp]),
    "gfq_comm_free": (None, [vp]),
    "gfq_echelonize_dist": (I, [vp, U32, vp, I64, I64, U64, _P(Options), I, vpp]),
    "gfq_dist_plan": (I, [U64, U64, U64, I, I, c_i32p, c_u64p, c_i32p, c_u64p]),
}


def load(path: str = LIB_PATH):
    if not os.path.exists(path):
        raise RuntimeError(
            f"libgfq.so not built at {path}: run __graft_entry__.build() "
            "(the B200 path has no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in PROTOS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def header_symbols(path: str = HEADER):
    """Function names declared in include/gfq.h."""
    import re
    txt = open(path).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(gfq_\w+)\s*\(", txt, re.M)))
