"""The reference's OWN unit tests, compiled unmodified against the drop-in.

/root/reference/proj/tests/test_grid.cpp, test_func2d.cpp and test_layer.cpp
are compiled as they are (no edit, no copy) with `-I tests/cpp/refshim`:
"lmkan/*.hpp" there alias include/lmkan_b200/lmkan.hpp with
`namespace lmkan = lmkan_b200;`, and catch_amalgamated.hpp is a minimal
Catch2-compatible harness (the reference's tolerances untouched). The binaries
are built by __graft_entry__.build() where /root/reference exists and travel
to the GPU box prebuilt (tests/cpp/_ref/).

test_grid / test_func2d exercise the host-side API (grid, thresholds,
interval_index, preamble, RandomStream, Func2D, eval2d, grad2d): CPU.
test_layer runs lmkan_forward / lmkan_backward on the GPU; its forward checks
compare at 1e-12 .. 1e-14 and finite differences at h = 1e-6, so it runs the
layers at reference precision (LMKAN_B200_PRECISION=fp64: the exact kernel,
bit-identical to the reference forward). At the default fp32 precision 3 of
its 9 cases fail on those fp64 tolerances, as expected of an fp32 forward.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_ref")


def _run(name, env=None):
    path = os.path.join(BIN, name)
    if not os.path.exists(path):
        import __graft_entry__ as g
        g.build_cpp_tests()
    if not os.path.exists(path):
        pytest.skip(f"{name}: reference sources absent and no prebuilt binary")
    r = subprocess.run([path], capture_output=True, text=True, timeout=600, env={**os.environ, **(env or {})})
    assert r.returncode == 0, r.stdout + r.stderr[-4000:]
    assert " 0 failures" in r.stdout
    return r.stdout


@pytest.mark.parametrize("name", ["test_grid", "test_func2d"])
def test_reference_host_unit_tests(name):
    _run(name)


@pytest.mark.gpu
def test_reference_layer_unit_tests_at_reference_precision():
    out = _run("test_layer", {"LMKAN_B200_PRECISION": "fp64"})
    assert out.startswith("9 test cases (0 failed)")
