"""The reference-side C++ drop-in (integration/gfrref_b200.cpp): its
gfrref_b200::echelonize, called with reference gfrref::Matrix / FieldSpec /
EchelonizeOptions values, returns an EchelonOutput equal field by field to
the reference's own gfrref::echelonize, and the reference's gfrref::verify
accepts it (tests/cpp/test_dropin.cpp, built by integration/Makefile against
/root/reference's headers and the reference library in oracle/_ref)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "integration", "_build", "test_dropin")


@pytest.mark.skipif(not os.path.exists(BIN), reason="integration/_build/test_dropin not built")
@pytest.mark.parametrize("mode", ["quick", "full"])
def test_cpp_dropin_matches_reference(mode):
    r = subprocess.run([BIN, mode], capture_output=True, text=True, timeout=900)
    lines = r.stdout.splitlines()
    bad = [ln for ln in lines if ln.startswith("FAIL")]
    assert r.returncode == 0 and not bad, "\n".join(bad + [r.stderr[-2000:]])
    assert sum(ln.startswith("PASS") for ln in lines) >= (24 if mode == "quick" else 26)
