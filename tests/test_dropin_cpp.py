"""GPU: run the C++ drop-in test program (tests/cpp/test_dropin.cpp), which
exercises include/lmkan_b200/lmkan.hpp exactly like the reference's
test_layer.cpp forward cases."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "test_dropin")


@pytest.mark.gpu
def test_cpp_dropin_api():
    if not os.path.exists(BIN):
        import __graft_entry__ as g
        g.build_cpp_tests()
    r = subprocess.run([BIN, os.path.join(ROOT, "tests", "golden", "lmk1")], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


def test_cpp_dropin_builds():
    """The drop-in header compiles against the C-ABI (no GPU needed)."""
    import __graft_entry__ as g
    g.build_cpp_tests()
    assert os.path.exists(BIN)
