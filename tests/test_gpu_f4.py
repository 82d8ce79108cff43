"""GPU parity of K1f, the FP4 tensor-core contraction (tcgen05.mma
kind::mxf4, gf_mad_f4.cu) for p in {2, 3, 5, 7}, against the CPU oracle's
mul_add_kernel restatement (oracle.mad; reference src/matrix.cpp:81-133).
Integer work: bit-exact.  The fp32 accumulation is exact while
|sum| <= ((p-1)/2)^2.k < 2^24; the extreme-value cases push the sums to
their largest magnitude."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

F4_PRIMES = [2, 3, 5, 7]


@pytest.fixture(scope="module")
def G():
    from paper_1806_04211_b200 import gfrref
    gfrref.lib()
    return gfrref


def rnd(p, m, n, seed):
    return oracle.random_matrix(p, m, n, seed)


def f4_launches(G):
    return G.profile_take_kinds()["k1_f4"][0]


@pytest.mark.parametrize("p", F4_PRIMES)
def test_f4_random_and_ragged(G, p):
    G.set_mad_policy(3)
    G.profile(True)
    G.profile_take_kinds()
    try:
        f = G.FieldSpec(p)
        for t, (m, k, n) in enumerate([(7, 5, 9), (128, 128, 192), (129, 257, 255), (500, 499, 1000),
                                       (1, 1, 1), (300, 64, 17), (64, 1024, 512), (256, 100, 513),
                                       (1000, 3000, 700), (128, 65, 384)]):
            a, b, c = rnd(p, m, k, 10 * t + 1), rnd(p, k, n, 10 * t + 2), rnd(p, m, n, 10 * t + 3)
            np.testing.assert_array_equal(G.mad(f, c, a, b).numpy(), oracle.mad(p, a, b, c))
            np.testing.assert_array_equal(G.mul(f, a, b).numpy(), oracle.mad(p, a, b))
        assert f4_launches(G) >= 20
    finally:
        G.profile(False)
        G.set_mad_policy(0)


@pytest.mark.parametrize("p", F4_PRIMES)
def test_f4_extreme_sums(G, p):
    """Largest |sum|: every entry the residue of largest symmetric magnitude
    (p = 2: all ones), with the same sign (positive sum) and with opposite
    signs on A and B (negative sum), up to deep K."""
    h = 1 if p == 2 else (p - 1) // 2
    G.set_mad_policy(3)
    try:
        f = G.FieldSpec(p)
        for k in (4096, 65536, 200000):
            for sa, sb in ((h, h), (h, p - h)):
                a = np.full((130, k), sa, np.uint8)
                b = np.full((k, 200), sb, np.uint8)
                c = np.full((130, 200), p - 1, np.uint8)
                want = (np.int64(sa) * sb * k + (p - 1)) % p
                got = G.mad(f, c, a, b).numpy()
                assert (got == want).all(), (p, k, sa, sb, np.unique(got))
    finally:
        G.set_mad_policy(0)


def test_f4_matches_i8_large(G):
    """A cfg-sized product on both tensor-core paths, device-resident."""
    for p in (2, 7):
        f = G.FieldSpec(p)
        A = G.random_matrix(f, 2048, 4096, 11)
        B = G.random_matrix(f, 4096, 3000, 12)
        C = G.random_matrix(f, 2048, 3000, 13)
        outs = []
        for pol in (2, 3):
            G.set_mad_policy(pol)
            try:
                outs.append(G.mad(f, C, A, B).numpy())
            finally:
                G.set_mad_policy(0)
        np.testing.assert_array_equal(outs[0], outs[1])


def test_f4_not_for_other_fields(G):
    """p = 11, 251: the policy falls back to kind::i8 (E2M1 cannot hold the residues)."""
    G.set_mad_policy(3)
    G.profile(True)
    G.profile_take_kinds()
    try:
        for p in (11, 251):
            f = G.FieldSpec(p)
            a, b = rnd(p, 256, 512, 1), rnd(p, 512, 384, 2)
            np.testing.assert_array_equal(G.mul(f, a, b).numpy(), oracle.mad(p, a, b))
        assert f4_launches(G) == 0
    finally:
        G.profile(False)
        G.set_mad_policy(0)


@pytest.mark.parametrize("env", ["GFQ_F4_CLUSTER=1", "GFQ_F4_CLUSTER=4", "GFQ_F4_CLUSTER=12",
                                 "GFQ_K1_MAX_WAVES=1"])
def test_f4_launch_variants(env):
    """The non-default operand-sharing cluster shapes and row-piece launches
    (GFQ_K1_MAX_WAVES; env settings are read once per process) on the
    ragged, extreme and large cases, in a child process."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    k, v = env.split("=")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(root, "tests", "test_gpu_f4.py"), "-k",
                        "random_and_ragged or extreme or large"],
                       env=dict(os.environ, **{k: v}), cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
