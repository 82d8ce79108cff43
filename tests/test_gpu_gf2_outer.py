"""GPU parity of the two-level GF(2) ECH whose outer panels are factorized by
one cluster launch each (ech_gf2_outer.cu) at the cfg5s diagonal-block size
and on the shapes that stress its pivot search: windows without candidates
(far pivots), free columns, dependent rows.  The reference's own ech on an
8192^2 block takes minutes, so the large cases compare against the split
path (mode 0/3), which test_ech_gf2_split_vs_reference pins to the reference
on smaller blocks; the smaller cases here compare with the reference
directly."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    from paper_1806_04211_b200 import gfrref
    gfrref.lib()
    return gfrref


def both(G, H):
    f = G.FieldSpec(2)
    outs = []
    try:
        for mode in (4, 3):
            G.set_ech_mode(mode)
            outs.append(G.ech(f, H))
    finally:
        G.set_ech_mode(0)
    return outs


def same(a, b):
    assert a.rank() == b.rank()
    assert list(a.rho.members) == list(b.rho.members) and list(a.gamma.members) == list(b.gamma.members)
    for key in "MKR":
        np.testing.assert_array_equal(getattr(a, key).numpy(), getattr(b, key).numpy())


def matches_reference(e, H):
    want = oracle.ref_ech(2, H)
    assert e.rank() == want["rank"]
    assert list(e.rho.members) == list(want["rho"]) and list(e.gamma.members) == list(want["gamma"])
    for key in "MKR":
        np.testing.assert_array_equal(getattr(e, key).numpy(), want[key])


@pytest.mark.parametrize("case", ["square8192", "deficient8192", "tall8192x3000", "wide4096x8192"])
def test_gf2_outer_large_vs_split(G, case):
    f = G.FieldSpec(2)
    if case == "square8192":
        H = G.random_matrix(f, 8192, 8192, 1).numpy()
    elif case == "deficient8192":
        H = G.random_matrix(f, 8192, 8192, 2).numpy()
        rng = np.random.default_rng(3)
        H[6000:6100] = H[rng.integers(0, 6000, 100)] ^ H[rng.integers(0, 6000, 100)]
        H[:, 5000:5040] = 0
    elif case == "tall8192x3000":
        H = G.random_matrix(f, 8192, 3000, 4).numpy()
    else:
        H = G.random_matrix(f, 4096, 8192, 5).numpy()
    a, b = both(G, H)
    same(a, b)


@pytest.mark.parametrize("case", ["window_miss", "free_cols", "dependent", "ragged"])
def test_gf2_outer_vs_reference(G, case):
    rng = np.random.default_rng(11)
    if case == "window_miss":
        # the first 1500 rows are zero in the first 96 columns: every early
        # column's pivot is a far row below the 64-row window
        H = oracle.random_matrix(2, 2500, 700, 21)
        H[:1500, :96] = 0
    elif case == "free_cols":
        H = oracle.random_matrix(2, 1800, 900, 22)
        H[:, rng.choice(900, 200, replace=False)] = 0
    elif case == "dependent":
        H = oracle.random_matrix(2, 2000, 1200, 23)
        H[1000:1600] = H[rng.integers(0, 1000, 600)] ^ H[rng.integers(0, 1000, 600)]
    else:
        H = oracle.random_matrix(2, 1333, 517, 24)
    e, s = both(G, H)
    matches_reference(e, H)
    same(e, s)
