"""CPU: pin the oracle before trusting it.

1. The C restatement (oracle/lmkan_oracle.c) against the reference's own
   known-answer tests, restated from test_grid.cpp / test_layer.cpp.
2. The C restatement against golden vectors produced by the reference itself
   (tests/golden/make_golden.py over oracle/_ref), bit for bit.
3. The C restatement against oracle/_ref on fresh random inputs (when the
   reference build is present).
4. The threshold tables that make cell indices bit-exact: exhaustively for
   G=16 over all 2^32 fp32 patterns, windowed around every threshold for the
   other grid sizes.
"""
import math
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden", "golden.npz")


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


# ---- 1. reference KATs (test_grid.cpp / test_layer.cpp) -------------------

def test_sigma_kats(port):  # test_grid.cpp:34-48
    assert port.sigma(0.0) == 0.5
    assert port.sigma(-math.log(2.0)) == pytest.approx(0.25, rel=1e-15)
    assert port.sigma(0.1) == pytest.approx(0.5475812909820202, rel=1e-15)
    assert math.isnan(port.sigma(float("nan")))
    xs = np.arange(-30.0, 30.0, 0.5)
    s = [port.sigma(x) for x in xs]
    assert all(b > a for a, b in zip(s, s[1:]))


def test_build_grid_kats(port):  # test_grid.cpp:65-85
    ln2 = math.log(2.0)
    pts, inv = port.build_grid(4)
    np.testing.assert_allclose(pts, [-2 * ln2, -ln2, 0.0, ln2, 2 * ln2], rtol=1e-15)
    assert pts[2] == 0.0
    assert inv[1 * 4 + 1] == pytest.approx(1.0 / (ln2 * ln2), rel=1e-14)
    p3, _ = port.build_grid(3)
    assert p3[0] == 2 * p3[1] - p3[2] and p3[3] == 2 * p3[2] - p3[1]
    for bad in (2, 0):
        with pytest.raises(ValueError):
            port.build_grid(bad)


@pytest.mark.parametrize("G", [3, 4, 5, 12, 13, 40])
def test_grid_invariants(port, G):  # test_grid.cpp:87-106
    pts, inv = port.build_grid(G)
    assert (np.diff(pts) > 0).all()
    assert (pts == -pts[::-1]).all()
    if G % 2 == 0:
        assert pts[G // 2] == 0.0
    assert np.isfinite(inv).all() and (inv > 0).all()
    if G >= 4:
        assert pts[2] - pts[1] == pytest.approx(math.log(2.0), rel=1e-14)


def test_interval_index_kats(port):  # test_grid.cpp:108-114
    assert port.interval_index(4, 0.1) == 2
    assert port.interval_index(4, -100.0) == 0
    assert port.interval_index(4, 100.0) == 3
    assert port.interval_index(4, 1e308) == 3
    assert port.interval_index(4, float("nan")) == 0


def test_interval_index_vs_binary_search(port):  # test_grid.cpp:116-132
    rng = np.random.default_rng(42)
    for G in (3, 4, 12, 40):
        pts, _ = port.build_grid(G)
        xs = np.concatenate([rng.standard_normal(5000), np.tan(np.pi * (rng.random(5000) - 0.5))])
        for x in xs:
            assert port.interval_index(G, x) == np.searchsorted(pts[1:G], x, side="right")


def test_preamble_kats(port):  # test_grid.cpp:166-195
    pts, _ = port.build_grid(4)
    i1, i2, w = port.locate(4, np.array([[pts[1], pts[1]]]))
    assert (i1[0, 0], i2[0, 0]) == (1, 1)
    np.testing.assert_allclose(w[0, 0], [1, 0, 0, 0], atol=1e-14)
    m1, m2 = 0.5 * (pts[1] + pts[2]), 0.5 * (pts[2] + pts[3])
    i1, i2, w = port.locate(4, np.array([[m1, m2]]))
    assert (i1[0, 0], i2[0, 0]) == (1, 2)
    np.testing.assert_allclose(w[0, 0], [0.25] * 4, atol=1e-14)
    i1, _, w = port.locate(4, np.array([[-10.0, 0.0]]))
    assert i1[0, 0] == 0 and w[0, 0, 1] < 0.0 < 1.0 < w[0, 0, 0]
    assert w[0, 0].sum() == pytest.approx(1.0, abs=1e-12)


def test_partition_of_unity(port):  # test_grid.cpp:197-219
    rng = np.random.default_rng(7)
    for G in (3, 4, 12, 40):
        X = rng.standard_normal((2000, 2))
        _, _, w = port.locate(G, X)
        assert np.abs(w.sum(-1) - 1.0).max() <= 1e-12


def test_forward_kats(port):  # test_layer.cpp:50-99, 112-145 (fp64 oracle semantics)
    rng = np.random.default_rng(11)
    # zero table -> zero output; gamma scales
    P = np.zeros((5, 5, 2, 3))
    assert (port.forward(4, P, rng.standard_normal((16, 4)), 1.0) == 0).all()
    # single function == direct bilinear evaluation (eval2d, func2d.hpp:51-56)
    G = 5
    P = rng.standard_normal((G + 1, G + 1, 1, 1))
    X = rng.standard_normal((64, 2))
    Y = port.forward(G, P, X, 1.0)
    i1, i2, w = port.locate(G, X)
    f = P[:, :, 0, 0]
    want = [w[r, 0, 0] * f[i1[r, 0], i2[r, 0]] + w[r, 0, 2] * f[i1[r, 0], i2[r, 0] + 1] +
            w[r, 0, 1] * f[i1[r, 0] + 1, i2[r, 0]] + w[r, 0, 3] * f[i1[r, 0] + 1, i2[r, 0] + 1] for r in range(64)]
    np.testing.assert_allclose(Y[:, 0], want, rtol=0, atol=1e-14)
    # linear sheets: f_qp = A x1 + B x2 + C is reproduced exactly by bilinear
    # interpolation, also on the extrapolating edge cells (test_layer.cpp:112-145)
    G, n_in, n_out = 4, 8, 3
    pts, _ = port.build_grid(G)
    A, Bm, Cm = (rng.standard_normal((n_out, n_in // 2)) for _ in range(3))
    P = (A.T[None, None] * pts[:, None, None, None] + Bm.T[None, None] * pts[None, :, None, None]
         + Cm.T[None, None])
    X = rng.standard_normal((32, n_in)) * 2.0
    Y = port.forward(G, P, X, 0.6)
    want = 0.6 * (X[:, 0::2] @ A.T + X[:, 1::2] @ Bm.T + Cm.sum(1))
    np.testing.assert_allclose(Y, want, rtol=0, atol=1e-10)


# ---- 2. golden vectors from the reference itself --------------------------

def test_golden_grids_and_locate(port, gold):
    Gs = sorted({int(k.split("_")[1][1:]) for k in gold.files if k.startswith("grid_")})
    assert Gs
    for G in Gs:
        pts, inv = port.build_grid(G)
        assert np.array_equal(pts, gold[f"grid_G{G}_points"]) and np.array_equal(inv, gold[f"grid_G{G}_inv"])
        i1, i2, w = port.locate(G, gold[f"loc_G{G}_X"])
        assert np.array_equal(i1, gold[f"loc_G{G}_i1"]) and np.array_equal(i2, gold[f"loc_G{G}_i2"])
        assert np.array_equal(w, gold[f"loc_G{G}_w"], equal_nan=True)


def test_golden_thresholds(port, gold):
    for k in gold.files:
        if k.startswith("thr_") and k.endswith("_f32"):
            G = int(k.split("_")[1][1:])
            assert np.array_equal(port.thresholds_f32(G), gold[k])
            assert np.array_equal(port.thresholds_f64(G), gold[k.replace("f32", "f64")])


def test_golden_forward(port, gold):
    k = 0
    while f"fwd_{k}_shape" in gold.files:
        n_in, n_out, G, rows = gold[f"fwd_{k}_shape"]
        Y = port.forward(int(G), gold[f"fwd_{k}_P"].astype(np.float64), gold[f"fwd_{k}_X"].astype(np.float64),
                         float(gold[f"fwd_{k}_gamma"]), threads=2)
        assert np.array_equal(Y, gold[f"fwd_{k}_Y"]), k  # bitwise: same fp64 operation order
        k += 1
    assert k >= 5


# ---- 3. restatement vs the live reference build ---------------------------

def test_port_matches_reference_build(port):
    import pyoracle
    try:
        ref = pyoracle.Ref()
    except (FileNotFoundError, OSError):
        pytest.skip("oracle/_ref not built (no /root/reference here)")
    rng = np.random.default_rng(3)
    for G in (3, 8, 16, 28, 32):
        X = np.concatenate([rng.standard_normal((200, 16)), np.tan(np.pi * (rng.random((200, 16)) - 0.5))])
        for a, b in zip(port.locate(G, X), ref.locate(G, X)):
            assert np.array_equal(a, b)
        P = rng.standard_normal((G + 1, G + 1, 8, 9))
        assert np.array_equal(port.forward(G, P, X, 0.7, threads=4), ref.forward(G, P, X, 0.7, workers=3))


# ---- 4. thresholds -> bit-exact cell indices ------------------------------

def _key32(bits):
    return bits


@pytest.mark.parametrize("G", [3, 5, 8, 13, 16, 28, 32, 40, 64])
def test_thresholds_windows(port, G):
    """#{k : x >= t_k} == interval_index(x) for every fp32 within 2^16 ulps of
    each threshold, all subnormal/tiny magnitudes, both infinities and NaNs,
    and a 1/65537 stride over all 2^32 patterns."""
    t = port.thresholds_f32(G)
    ranges = [(0x00000000, 0x0001FFFF), (0x80000000, 0x8001FFFF), (0x7F7F0000, 0x7FFFFFFF),
              (0xFF7F0000, 0xFFFFFFFF)]
    for tk in t:
        b = int(np.array([tk], np.float32).view(np.uint32)[0])
        ranges.append((max(b - 65536, 0), min(b + 65536, 0xFFFFFFFF)))
    for lo, hi in ranges:
        assert port.verify_thresholds_f32(G, t, lo, hi, threads=8) == 0, (G, hex(lo), hex(hi))
    # stride sample over everything
    bits = np.arange(0, 2 ** 32, 65537, dtype=np.uint64).astype(np.uint32)
    xs = bits.view(np.float32)
    cnt = (xs[:, None] >= t[None, :]).sum(1)
    ref = np.array([port.interval_index(G, float(x)) for x in xs])
    assert np.array_equal(cnt, ref)


def test_thresholds_exhaustive_G16(port):
    """All 2^32 fp32 bit patterns (about 15 s on 8 cores)."""
    t = port.thresholds_f32(16)
    assert port.verify_thresholds_f32(16, t, 0, 0xFFFFFFFF, threads=os.cpu_count() or 8) == 0


def test_backward_port_bitwise_vs_reference():
    """The C restatement of lmkan_backward (lmko_backward) is bit-identical to
    the reference's (layer.hpp:141-202) at workers = 1, dP += semantics included."""
    import pyoracle
    try:
        ref = pyoracle.Ref()
    except (FileNotFoundError, OSError):
        pytest.skip("oracle/_ref not built")
    port = pyoracle.Port()
    for (n_in, n_out, G, rows) in [(2, 1, 4, 16), (6, 5, 3, 40), (8, 6, 12, 33), (12, 16, 28, 64)]:
        rng = np.random.default_rng(G + n_in)
        P = rng.standard_normal((G + 1, G + 1, n_in // 2, n_out))
        X = rng.standard_normal((rows, n_in)) * 1.5
        X[::5, 0] = 80.0
        dY = rng.standard_normal((rows, n_out))
        dP0 = rng.standard_normal(P.shape)
        a = ref.backward(G, P, X, dY, 0.7, dP0=dP0, workers=1)
        b = port.backward(G, P, X, dY, 0.7, dP0=dP0)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
