"""GPU tests of the text formats and the cmd_ech drop-in:
GFMAT / SELECTS / TRANSFORM files written from the B200 outputs must be
byte-identical to the reference's own writers (oracle/_ref, compiled from
/root/reference) on the same seeded inputs; the CLI keeps the reference's
exit codes (include/gfrref/cli.hpp:10-13)."""
import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
needs_ref = pytest.mark.skipif(not os.path.exists(oracle.REF_ECH), reason="oracle/_ref/ref_ech not built")


@pytest.fixture(scope="module")
def G():
    from paper_1806_04211_b200 import gfrref
    gfrref.lib()
    return gfrref


def make(p, m, n, kind, seed):
    if kind == "random":
        return oracle.random_matrix(p, m, n, seed)
    if kind == "product":
        return oracle.random_product_matrix(p, m, n, min(m, n) // 2, seed)
    return np.zeros((m, n), np.uint8)


def read(path):
    with open(path, "rb") as fh:
        return fh.read()


@needs_ref
@pytest.mark.parametrize("p,m,n,block,kind,wt", [
    (3, 6, 6, 3, "random", True), (2, 130, 97, 32, "random", True), (7, 90, 120, 40, "product", True),
    (251, 64, 64, 32, "random", True), (5, 50, 70, 16, "product", False), (3, 20, 30, 8, "zero", True),
])
def test_files_byte_identical_to_reference(G, tmp_path, p, m, n, block, kind, wt):
    from paper_1806_04211_b200 import cli
    C = make(p, m, n, kind, 3)
    src = str(tmp_path / "in.gfmat")
    oracle.ref_write_gfmat(p, C, src)
    G.write_gfmat_file(str(tmp_path / "in_ours.gfmat"), G.FieldSpec(p), C)
    assert read(src) == read(str(tmp_path / "in_ours.gfmat"))
    rc, outp = oracle.ref_cli("ech", src, block, 2, int(wt), tmp_path / "r_ref", tmp_path / "s_ref",
                              tmp_path / "t_ref" if wt else "-")
    assert rc == 0
    args = ["ech", "--in", src, "--out-r", str(tmp_path / "r"), "--out-selects", str(tmp_path / "s"),
            "--block", str(block), "--threads", "2"]
    args += ["--out-t", str(tmp_path / "t")] if wt else ["--no-transform"]
    assert cli.main(args) == 0
    assert outp.strip().startswith("rank ")
    assert read(str(tmp_path / "r")) == read(str(tmp_path / "r_ref"))
    assert read(str(tmp_path / "s")) == read(str(tmp_path / "s_ref"))
    if wt:
        assert read(str(tmp_path / "t")) == read(str(tmp_path / "t_ref"))


def test_gfmat_roundtrip_and_errors(G, tmp_path):
    C = oracle.random_matrix(7, 33, 17, 9)
    path = str(tmp_path / "c.gfmat")
    G.write_gfmat_file(path, G.FieldSpec(7), C)
    f, M = G.read_gfmat_file(path)
    assert f.p == 7
    np.testing.assert_array_equal(M.numpy(), C)
    bad = {
        "header": "GFMAT v2\nfield p=7 k=1\nrows=1 cols=1\n0\n",
        "entry": "GFMAT v1\nfield p=7 k=1\nrows=1 cols=2\n0 7\n",
        "count": "GFMAT v1\nfield p=7 k=1\nrows=2 cols=2\n0 1\n1\n",
        # GF(p^k) files load (tests/test_gpu_ext.py, test_gpu_wide.py); these do not
        "reducible": "GFMAT v1\nfield p=2 k=2 modulus=1,0,1\nrows=1 cols=1\n0\n",
        "range": "GFMAT v1\nfield p=11 k=3 modulus=4,1,0,1\nrows=1 cols=1\n1331\n",
        "trailing": "GFMAT v1\nfield p=3 k=1\nrows=1 cols=1\n2\nextra\n",
    }
    for what, text in bad.items():
        fp = str(tmp_path / f"{what}.gfmat")
        with open(fp, "w") as fh:
            fh.write(text)
        with pytest.raises(ValueError) as ei:
            G.read_gfmat_file(fp)
        assert fp in str(ei.value), what
    # GF(11^3) (the reference's own test field, q = 1331) loads, u32 elements
    fp = str(tmp_path / "w.gfmat")
    with open(fp, "w") as fh:
        fh.write("GFMAT v1\nfield p=11 k=3 modulus=4,1,0,1\nrows=1 cols=2\n0 1330\n")
    f, M = G.read_gfmat_file(fp)
    assert (f.p, f.k, f.q) == (11, 3, 1331) and M.esize == 4 and M.numpy().tolist() == [[0, 1330]]


def test_cli_exit_codes(G, tmp_path, capsys):
    from paper_1806_04211_b200 import cli
    C = oracle.random_product_matrix(3, 40, 40, 25, 4)
    path = str(tmp_path / "c.gfmat")
    G.write_gfmat_file(path, G.FieldSpec(3), C)
    assert cli.main(["rank", "--in", path, "--block", "16"]) == 0
    assert capsys.readouterr().out.strip() == "rank 25"
    assert cli.main(["ech", "--in", path, "--no-transform", "--out-t", str(tmp_path / "t")]) == 2
    assert cli.main(["ech", "--in", str(tmp_path / "missing.gfmat")]) == 2
    with open(str(tmp_path / "bad.gfmat"), "w") as fh:
        fh.write("not a matrix\n")
    assert cli.main(["ech", "--in", str(tmp_path / "bad.gfmat")]) == 2
    assert cli.main(["ech", "--in", path, "--block", "0"]) == 2
