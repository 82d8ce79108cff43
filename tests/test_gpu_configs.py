"""BASELINE.json configs at full size (configs[1..4], configs[4] as its
1-GPU 65536^2 leading case).

* cfg2a / cfg2b / cfg3: bit-exact against the reference's own blocked
  echelonize (oracle/_ref, compiled from /root/reference, all host threads)
  on the same seeded input: rank, pivot columns, row selects, every R /
  T_M / T_K block.
* cfg4 / cfg5s (too slow for the CPU reference in a test): the defining
  identity T.C = E checked on the device (gfq_verify exact / Freivalds),
  the echelon shape of R, and block-size independence of the canonical
  outputs on a leading submatrix.
"""
import numpy as np
import pytest

import oracle

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def G():
    from paper_1806_04211_b200 import gfrref
    gfrref.lib()
    return gfrref


def run(G, name, threads=4, with_transform=True):
    from paper_1806_04211_b200 import workloads
    cfg = workloads.CONFIGS[name]
    f = G.FieldSpec(cfg["p"])
    C = workloads.build(G, name)
    out = G.echelonize(C, f, G.EchelonizeOptions(block=cfg["block"], threads=threads,
                                                 with_transform=with_transform))
    return cfg, f, C, out


def same_as_reference(out, ref):
    assert out.rank == ref.rank
    for j in range(ref.b):
        assert list(out.upsilon[j].members) == ref.upsilon(j).tolist(), ("upsilon", j)
        for l in range(j, ref.b):
            np.testing.assert_array_equal(out.block(0, j, l).numpy(), ref.block(0, j, l), err_msg=f"R {j},{l}")
        for h in range(ref.a):
            np.testing.assert_array_equal(out.block(1, j, h).numpy(), ref.block(1, j, h), err_msg=f"TM {j},{h}")
    for i in range(ref.a):
        assert list(out.varrho[i].members) == ref.varrho(i).tolist(), ("varrho", i)
        for h in range(i + 1):
            np.testing.assert_array_equal(out.block(2, i, h).numpy(), ref.block(2, i, h), err_msg=f"TK {i},{h}")


@pytest.mark.skipif(oracle.ref is None, reason="oracle/_ref not built")
@pytest.mark.parametrize("name", ["cfg2a", "cfg2b", "cfg3"])
def test_config_vs_reference_library(G, name):
    cfg, f, C, out = run(G, name)
    threads = max(1, oracle.ref.ref_hardware_concurrency())
    ref = oracle.ref_echelonize(cfg["p"], C.numpy(), cfg["block"], threads=threads)
    same_as_reference(out, ref)
    if name == "cfg2b":
        assert out.rank <= 4096 and len(out.upsilon[0].members) == 0
    if name == "cfg3":
        assert out.rank == 10000
    ok, diag, _ = G.verify(C, out, "freivalds")
    assert ok, diag


def test_cfg2a_exact_identity(G):
    cfg, f, C, out = run(G, "cfg2a")
    ok, diag, checked = G.verify(C, out, "exact")
    assert ok and checked == "exact", diag


def test_cfg4_identity_and_block_independence(G):
    cfg, f, C, out = run(G, "cfg4")
    assert out.rank == cfg["m"]  # a random 32768^2 GF(251) matrix is invertible w.h.p.
    ok, diag, checked = G.verify(C, out, "exact")
    assert ok and checked == "exact", diag
    # the canonical outputs do not depend on the block size: a 4096 x 6144
    # leading slab at block 4096 vs block 1024, assembled R and T compared.
    sub = G.Matrix.from_numpy(C.numpy()[:4096, :6144])
    o1 = G.echelonize(sub, f, G.EchelonizeOptions(block=4096, threads=4))
    o2 = G.echelonize(sub, f, G.EchelonizeOptions(block=1024, threads=4))
    assert o1.rank == o2.rank == 4096
    assert o1.global_upsilon() == o2.global_upsilon()
    np.testing.assert_array_equal(o1.assembled_R().numpy(), o2.assembled_R().numpy())
    np.testing.assert_array_equal(o1.materialize_transform().numpy(), o2.materialize_transform().numpy())


def test_cfg5s_identity(G):
    cfg, f, C, out = run(G, "cfg5s")
    ok, diag, checked = G.verify(C, out, "freivalds")
    assert ok and checked == "freivalds", diag
    assert out.rank >= cfg["m"] - 64  # a random GF(2) square matrix loses O(1) rank
