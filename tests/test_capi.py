"""CPU: the C-ABI library loads, exports every symbol include/lmkan_b200.h
declares, and its host-only entry points match the oracle; compute entry
points fail loudly (no CPU fallback) when no GPU is visible."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lmkan_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lmkan_b200_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import paper_2509_07103_b200 as pkg
    lib = ctypes.CDLL(pkg.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # and the Python binding binds exactly what the header declares
    from paper_2509_07103_b200._lib import _SIGS
    assert sorted(n for n, _, _ in _SIGS) == syms


def test_library_is_sm100a_cuda():
    import paper_2509_07103_b200 as pkg
    out = os.popen(f"cuobjdump --list-elf {pkg.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out


def test_build_grid_matches_golden_and_errors():
    import paper_2509_07103_b200 as pkg
    gold = np.load(os.path.join(ROOT, "tests", "golden", "golden.npz"))
    for G in (3, 4, 5, 8, 12, 13, 16, 20, 28, 32, 40):
        g = pkg.build_grid(G)
        assert np.array_equal(g.points, gold[f"grid_G{G}_points"])
        assert np.array_equal(g.inv_areas, gold[f"grid_G{G}_inv"])
        t64, t32 = pkg.thresholds(G)
        assert np.array_equal(t32, gold[f"thr_G{G}_f32"]) and np.array_equal(t64, gold[f"thr_G{G}_f64"])
    with pytest.raises(ValueError, match="G must be >= 3"):
        pkg.build_grid(2)
    with pytest.raises(ValueError, match="G must be >= 3"):
        pkg.thresholds(0)


def test_thresholds_reproduce_reference_index(port):
    """#{k: x >= t_k} with the PRODUCT's tables equals the oracle index on
    random and edge-case doubles (f64 path) and floats (f32 path)."""
    import paper_2509_07103_b200 as pkg
    rng = np.random.default_rng(5)
    for G in (3, 8, 16, 28, 32, 40, 64):
        t64, t32 = pkg.thresholds(G)
        xs = np.concatenate([rng.standard_normal(3000), np.tan(np.pi * (rng.random(3000) - 0.5)),
                             t64, np.nextafter(t64, -np.inf), np.nextafter(t64, np.inf),
                             [0.0, -0.0, -2.0 ** -54, -1e-300, np.inf, -np.inf, np.nan]])
        ref = np.array([port.interval_index(G, x) for x in xs])
        assert np.array_equal((xs[:, None] >= t64[None, :]).sum(1), ref)
        xf = xs.astype(np.float32)
        ref32 = np.array([port.interval_index(G, float(x)) for x in xf])
        assert np.array_equal((xf[:, None] >= t32[None, :]).sum(1), ref32)


def test_init_table_bit_identical_to_reference(port):
    import paper_2509_07103_b200 as pkg
    gold = np.load(os.path.join(ROOT, "tests", "golden", "golden.npz"))
    k = 0
    while f"init_{k}_args" in gold.files:
        n_in, n_out, G, seed, sc = gold[f"init_{k}_args"]
        P = pkg.init_table(int(n_in), int(n_out), int(G), int(seed), float(sc))
        assert np.array_equal(P, gold[f"init_{k}_P"])
        k += 1
    assert k == 4
    lay = pkg.init_layer(4, 3, 4, 123)
    assert lay.gamma == 0.0 and lay.P.shape == (5, 5, 2, 3) and lay.param_count() == 150
    assert not np.array_equal(lay.P, pkg.init_layer(4, 3, 4, 124).P)
    with pytest.raises(ValueError, match="n_in must be a positive even number"):
        pkg.init_layer(3, 2, 4, 0)
    with pytest.raises(ValueError, match="n_in must be a positive even number"):
        pkg.init_layer(0, 2, 4, 0)
    with pytest.raises(ValueError, match="n_out must be positive"):
        pkg.init_layer(4, 0, 4, 0)


def test_width_mismatch_raises_like_reference():
    import paper_2509_07103_b200 as pkg
    lay = pkg.init_layer(4, 2, 4, 5)
    with pytest.raises(ValueError, match="lmkan_forward: expected width 4, got 6"):
        pkg.lmkan_forward(lay, np.zeros((3, 6)))


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2509_07103_b200 as pkg
    with pytest.raises(pkg.LmkanError, match="no CPU fallback"):
        pkg.Layer.random(8, 8, 4)
    lay = pkg.init_layer(4, 3, 4, 1)
    lay.gamma = 1.0
    with pytest.raises(pkg.LmkanError):
        pkg.lmkan_forward(lay, np.zeros((2, 4)))


def test_product_does_not_reference_oracle():
    """The shipped package never imports, links or loads anything under oracle/."""
    pkgdir = os.path.join(ROOT, "paper_2509_07103_b200")
    for dp, _, fs in os.walk(pkgdir):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".hpp", ".h", ".cpp")):
                s = open(os.path.join(dp, f)).read()
                assert "pyoracle" not in s and "lmkan_oracle" not in s and "liblmkan_ref" not in s, f
    out = os.popen(f"ldd {os.path.join(pkgdir, 'lib', 'liblmkan_b200.so')}").read()
    assert "oracle" not in out and "lmkan_ref" not in out
