"""GPU: lmkan_backward (layer.hpp:141-202) on the B200 path.

Bar: dP and dX BIT-IDENTICAL to the reference's own lmkan_backward run with
the same worker count (oracle/_ref; the C restatement, pinned bitwise to the
reference at workers = 1 in tests/test_oracle.py, covers workers = 1 when the
reference build is absent), including the += semantics of dP; plus the
reference's own backward test cases (test_layer.cpp:147-226) restated.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t
    return t


@pytest.fixture(scope="module")
def pkg():
    import paper_2509_07103_b200 as p
    return p


def _case(n_in, n_out, G, rows, seed, xscale=1.5):
    rng = np.random.default_rng(seed)
    P = rng.standard_normal((G + 1, G + 1, n_in // 2, n_out)) / np.sqrt(n_in // 2)
    X = rng.standard_normal((rows, n_in)) * xscale
    dY = rng.standard_normal((rows, n_out))
    return P, X, dY


SHAPES = [(2, 1, 4, 64), (6, 5, 3, 64), (6, 5, 12, 200), (8, 6, 12, 33), (32, 32, 12, 1000), (12, 128, 28, 512),
          (64, 64, 8, 300)]


@pytest.mark.parametrize("n_in,n_out,G,rows", SHAPES)
def test_backward_bitwise_vs_reference(torch, pkg, oracle, n_in, n_out, G, rows):
    P, X, dY = _case(n_in, n_out, G, rows, seed=n_in * 31 + G)
    X[::7, 0] = 100.0        # far right edge cell (extrapolation)
    X[1::7, 1] = -100.0      # far left edge cell
    X[2::7, 0] = -1e-30      # tiny negative: cell G/2 (grid.hpp:72-75)
    gamma = 0.7
    dP0 = np.random.default_rng(1).standard_normal(P.shape)  # dP is added into
    layer = pkg.Layer.from_host(n_in, n_out, G, P, gamma)
    Pd = torch.from_numpy(P).cuda()
    Xd, dYd = torch.from_numpy(X).cuda(), torch.from_numpy(dY).cuda()
    import pyoracle
    have_ref = isinstance(oracle, pyoracle.Ref)
    for workers in ([1, 3, 0] if have_ref else [1]):
        w = workers or layer.backward_workers(rows)
        ref_dP, ref_dX = oracle.backward(G, P, X, dY, gamma, dP0=dP0, workers=w)
        got_dP, got_dX = layer.backward(Pd, Xd, dYd, dP=torch.from_numpy(dP0).cuda(), workers=workers)
        assert np.array_equal(got_dP.cpu().numpy(), ref_dP), workers
        assert np.array_equal(got_dX.cpu().numpy(), ref_dX), workers
        # host path, same bits
        h_dP, h_dX = layer.backward(P, X, dY, dP=dP0, workers=workers)
        assert np.array_equal(h_dP, ref_dP) and np.array_equal(h_dX, ref_dX)


def test_backward_deterministic(torch, pkg):
    """Bitwise run to run (test_layer.cpp:228-239)."""
    P, X, dY = _case(32, 48, 12, 3000, seed=5)
    layer = pkg.Layer.from_host(32, 48, 12, P, 0.9)
    Pd, Xd, dYd = (torch.from_numpy(a).cuda() for a in (P, X, dY))
    a = layer.backward(Pd, Xd, dYd)
    b = layer.backward(Pd, Xd, dYd)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


def test_zero_upstream_and_compact_support(torch, pkg):
    """test_layer.cpp:147-176: dY = 0 gives dP = dX = 0; one row touches
    exactly the four nodes of its cell."""
    P, X, dY = _case(4, 3, 4, 8, seed=13)
    layer = pkg.Layer.from_host(4, 3, 4, P, 0.5)
    dP, dX = layer.backward(P, X, np.zeros_like(dY))
    assert not dP.any() and not dX.any()
    P1 = np.random.default_rng(7).standard_normal((5, 5, 1, 1))
    one = pkg.Layer.from_host(2, 1, 4, P1, 1.0)
    dP, _ = one.backward(P1, np.array([[0.2, -0.4]]), np.array([[1.0]]), want_dx=False)
    assert np.count_nonzero(dP) == 4


def test_finite_differences(pkg, oracle):
    """test_layer.cpp:178-226: dP against central differences of the
    reference's fp64 forward (linear in P, tight); dX away from cell edges."""
    h = 1e-6
    rng = np.random.default_rng(14)
    for G in (3, 4):
        P, X, dY = _case(4, 3, G, 8, seed=1000 + G, xscale=1.0)
        gamma = 0.7
        layer = pkg.Layer.from_host(4, 3, G, P, gamma)
        dP, dX = layer.backward(P, X, dY)

        def loss(Pm, Xm):
            return float((oracle.forward(G, Pm, Xm, gamma) * dY).sum())
        flat = P.reshape(-1)
        for i in range(0, flat.size, 7):
            Pp, Pm = flat.copy(), flat.copy()
            Pp[i] += h
            Pm[i] -= h
            fd = (loss(Pp.reshape(P.shape), X) - loss(Pm.reshape(P.shape), X)) / (2 * h)
            assert abs(dP.reshape(-1)[i] - fd) <= 1e-6 * max(1.0, abs(fd))
        i1, i2, _ = oracle.locate(G, X)
        for r in range(X.shape[0]):
            for j in range(4):
                xp, xm = X.copy(), X.copy()
                xp[r, j] += h
                xm[r, j] -= h
                a, b = oracle.locate(G, xp[r:r + 1]), oracle.locate(G, xm[r:r + 1])
                if not (np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])):
                    continue  # stencil crosses a cell edge
                fd = (loss(P, xp) - loss(P, xm)) / (2 * h)
                assert abs(dX[r, j] - fd) <= 1e-6 * max(1.0, abs(fd))
    del rng


def test_backward_argument_errors(torch, pkg):
    P, X, dY = _case(4, 3, 4, 8, seed=2)
    layer = pkg.Layer.from_host(4, 3, 4, P, 1.0)
    Pd, Xd, dYd = (torch.from_numpy(a).cuda() for a in (P, X, dY))
    with pytest.raises(ValueError, match="lmkan_backward: expected width 3"):
        layer.backward(Pd, Xd, torch.zeros((8, 4), dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError, match="row counts differ"):
        layer.backward(Pd, Xd, dYd[:5].contiguous())
    sl = pkg.Layer.from_device(4, 3, 4, Pd.float(), 1.0, out_range=(0, 2))
    with pytest.raises(ValueError, match="output-sliced|coefficients"):
        sl.backward(Pd, Xd, dYd[:, :2].contiguous())


def test_backward_nonfinite_inputs_bitwise(torch, pkg, oracle):
    """NaN / +-inf / huge inputs: the same bit patterns as the reference
    (NaN propagation included), compared as raw 64-bit words."""
    P, X, dY = _case(8, 6, 12, 40, seed=99)
    X[0, 0], X[1, 1], X[2, 2], X[3, 3] = np.nan, np.inf, -np.inf, 1e300
    X[4, :] = np.nan
    layer = pkg.Layer.from_host(8, 6, 12, P, 0.8)
    ref_dP, ref_dX = oracle.backward(12, P, X, dY, 0.8, workers=1)
    got_dP, got_dX = layer.backward(P, X, dY, workers=1)
    assert np.array_equal(got_dP.view(np.uint64), ref_dP.view(np.uint64))
    assert np.array_equal(got_dX.view(np.uint64), ref_dX.view(np.uint64))


def test_backward_argument_checks(torch, pkg):
    """dP / P / X / dY are validated before any pointer reaches the C-ABI
    (a float32 or mis-sized dP would otherwise be written out of bounds)."""
    layer = pkg.Layer.random(8, 6, 5, seed=2)
    n = 6 * 6 * 4 * 6
    P = torch.zeros(n, dtype=torch.float64, device="cuda")
    X = torch.zeros((3, 8), dtype=torch.float64, device="cuda")
    dY = torch.zeros((3, 6), dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError, match="dP must be"):
        layer.backward(P, X, dY, dP=torch.zeros(n, dtype=torch.float32, device="cuda"))
    with pytest.raises(ValueError, match="size mismatch"):
        layer.backward(P, X, dY, dP=torch.zeros(n + 1, dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError, match="coefficients"):
        layer.backward(P[:-1], X, dY)
    with pytest.raises(ValueError, match="contiguous float64"):
        layer.backward(P, X.float(), dY)
    with pytest.raises(ValueError, match="expected width 8"):
        layer.backward(P.cpu().numpy(), np.zeros((3, 9)), np.zeros((3, 6)))
    with pytest.raises(ValueError, match="row counts differ"):
        layer.backward(P.cpu().numpy(), np.zeros((3, 8)), np.zeros((2, 6)))
    dP, dX = layer.backward(P, X, dY)
    assert dP.shape == P.shape and dX.shape == X.shape


def test_forward_argument_checks(torch, pkg):
    layer = pkg.Layer.random(8, 6, 5, seed=2)
    X = torch.zeros((3, 8), device="cuda")
    with pytest.raises(ValueError, match="contiguous CUDA"):
        layer.forward_into(torch.zeros((8, 3), device="cuda").t(), torch.empty((3, 6), device="cuda"))
    with pytest.raises(ValueError, match="Y must be"):
        layer.forward_into(X, torch.empty((3, 6), device="cuda", dtype=torch.float64))
    with pytest.raises(ValueError, match="dtype"):
        layer.forward_dests(X.double(), [0], 6, 0)
    with pytest.raises(ValueError, match="ld must be"):
        layer.forward_dests(X, [torch.empty((3, 6), device="cuda").data_ptr()], 5, 0)
