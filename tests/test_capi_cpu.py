"""CPU-side checks of the C ABI boundary: libgfq.so loads without a GPU,
exports every symbol include/gfq.h declares, host-only entry points
(ChopMatrix, index-set jobs) behave like the reference, and compute entry
points fail loudly (no CPU fallback) when no device is present."""
import ctypes
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def rawlib():
    from paper_1806_04211_b200 import _capi
    if not os.path.exists(_capi.LIB_PATH):
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "paper_1806_04211_b200", "csrc")], check=True)
    return _capi.load()


def test_exports_every_header_symbol(rawlib):
    from paper_1806_04211_b200 import _capi
    declared = _capi.header_symbols()
    assert len(declared) > 40
    out = subprocess.run(["nm", "-D", "--defined-only", _capi.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    # every declared symbol also has a ctypes prototype
    assert not [s for s in declared if s not in _capi.PROTOS]


def test_library_links_only_system_libs(rawlib):
    from paper_1806_04211_b200 import _capi
    out = subprocess.run(["ldd", _capi.LIB_PATH], capture_output=True, text=True).stdout
    assert "libcudart" not in out  # static runtime: travels as one file
    assert "not found" not in out


def test_kernels_compiled_for_sm100a(rawlib):
    from paper_1806_04211_b200 import _capi
    sass = subprocess.run(["cuobjdump", "-sass", _capi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", _capi.LIB_PATH], capture_output=True,
                                       text=True).stdout
    assert "UTCIMMA" in sass       # tcgen05.mma kind::i8
    assert "UTMALDG" in sass       # TMA tensor loads
    assert "LDTM" in sass          # tcgen05.ld (TMEM -> registers)


def test_chop_matches_reference_semantics(rawlib):
    # reference tests/test_chief.cpp:78-118
    from paper_1806_04211_b200 import gfrref as G
    cs = G.chop(6, 6, 3)
    assert cs.row_parts == [3, 3] and cs.col_parts == [3, 3]
    assert G.chop(7, 7, 3).row_parts == [3, 3, 1]
    assert G.chop(7, 7, 3, remainder_first=True).row_parts == [1, 3, 3]
    single = G.chop(5, 4, 256)
    assert single.row_parts == [5] and single.col_parts == [4]
    e = G.chop(0, 5, 2)
    assert e.a() == 0 and e.b() == 3
    with pytest.raises(ValueError):
        G.chop(4, 4, 0)


def test_no_cpu_fallback_without_device(rawlib):
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except Exception:
        pass
    assert rawlib.gfq_init(0) == 3  # GFQ_ERR_CUDA
    msg = rawlib.gfq_last_error().decode()
    assert "CUDA" in msg or "device" in msg
    h = ctypes.c_void_p()
    buf = (ctypes.c_uint8 * 4)()
    rc = rawlib.gfq_mat_upload(2, 2, ctypes.cast(buf, ctypes.POINTER(ctypes.c_uint8)), 2, ctypes.byref(h))
    assert rc == 3


def test_index_jobs_host_side(rawlib):
    """unh / mkr are O(alpha) host merges; they run without a device."""
    from paper_1806_04211_b200 import _capi

    def iset(u, mem):
        arr = (ctypes.c_uint32 * max(len(mem), 1))(*mem)
        h = ctypes.c_void_p()
        assert rawlib.gfq_iset_create(u, arr, len(mem), ctypes.byref(h)) == 0
        return h

    def get(h):
        u, n = ctypes.c_uint64(), ctypes.c_uint64()
        rawlib.gfq_iset_get(h, ctypes.byref(u), ctypes.byref(n), None)
        buf = (ctypes.c_uint32 * max(n.value, 1))()
        rawlib.gfq_iset_get(h, None, None, buf)
        return u.value, list(buf[: n.value])

    def bits(h):
        n = ctypes.c_uint64()
        rawlib.gfq_bits_get(h, ctypes.byref(n), None)
        buf = (ctypes.c_uint8 * max(n.value, 1))()
        rawlib.gfq_bits_get(h, None, buf)
        return list(buf[: n.value])

    rho, u = ctypes.c_void_p(), ctypes.c_void_p()
    # reference tests/test_jobs.cpp:236-245
    assert rawlib.gfq_unh(iset(9, [2, 5, 6]), iset(6, [0, 3, 5]), ctypes.byref(rho), ctypes.byref(u)) == 0
    assert get(rho) == (9, [0, 2, 4, 5, 6, 8])
    assert bits(u) == [1, 0, 1, 0, 0, 1]
    mk = ctypes.c_void_p()
    assert rawlib.gfq_mkr(iset(3, [0, 2]), iset(3, [0, 1, 2]), ctypes.byref(mk)) == 0
    assert bits(mk) == [1, 0, 1]
    assert rawlib.gfq_mkr(iset(4, [2]), iset(4, [0, 3]), ctypes.byref(mk)) == 1  # invalid_argument
    assert b"subset" in rawlib.gfq_last_error()
    assert rawlib.gfq_unh(iset(4, [0]), iset(4, [0]), ctypes.byref(rho), ctypes.byref(u)) == 1
