"""Reference-precision layers (lmkan_b200_layer_create_exact, csrc/exact.cu):
the forward is BIT-IDENTICAL to the reference's lmkan_forward (layer.hpp:108-134,
via oracle/_ref), compared as raw 64-bit words (NaN: same positions)."""
import numpy as np
import pytest

from test_parity_gpu import SHAPES, _inputs, _special_rows

pytestmark = pytest.mark.gpu


def _assert_bits(Y, ref):
    Y = np.ascontiguousarray(Y, np.float64)
    ref = np.ascontiguousarray(ref, np.float64)
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(Y), nan), "NaN positions differ"
    yb, rb = Y.view(np.uint64)[~nan], ref.view(np.uint64)[~nan]
    bad = np.flatnonzero(yb != rb)
    assert bad.size == 0, f"{bad.size} outputs differ, first {Y[~nan][bad[0]]!r} vs {ref[~nan][bad[0]]!r}"


@pytest.mark.parametrize("n_in,n_out,G,rows", SHAPES)
def test_exact_forward_bitwise(torch, pkg, oracle, n_in, n_out, G, rows):
    P, X = _inputs(torch, n_in, n_out, G, rows, seed=5 * n_in + G)
    P = P.astype(np.float64) * (1 + 1e-9)  # not fp32-representable: the fp64 table is used as is
    X = np.concatenate([X.astype(np.float64) * 1.37, _special_rows(n_in, G, pkg).astype(np.float64)])
    X[np.isfinite(X) & (np.abs(X) > 1e6)] = 1e6
    layer = pkg.Layer.from_host(n_in, n_out, G, P, 0.9, precision=64)
    assert layer.plan(X.shape[0])["mode"] == "exact"
    ref = oracle.forward(G, P, X, 0.9)
    _assert_bits(layer.forward(torch.from_numpy(X).cuda()).cpu().numpy(), ref)
    # host entry (row chunks, pageable staging; fp64 Y is NOT narrowed for exact layers)
    _assert_bits(layer.forward_host(X), ref)


@pytest.mark.parametrize("n_in,n_out,G,rows,gamma", [
    (2, 1, 3, 77, 1.0), (6, 5, 12, 64, 0.8), (10, 7, 40, 333, 1.0), (12, 9, 64, 100, 0.5),
    (30, 100, 9, 777, 1.3), (8, 33, 28, 1025, 0.0), (64, 64, 8, 5000, 1.0), (6, 3, 200, 40, 1.1),
])
def test_exact_small_ragged_and_large_g(torch, pkg, oracle, n_in, n_out, G, rows, gamma):
    """Ragged output tiles, gamma = 0, every sheet width (OT 32 / 16 / 8) and
    the sheets-from-L2 variant (G = 64)."""
    rng = np.random.default_rng(n_in + G)
    P = rng.standard_normal((G + 1, G + 1, n_in // 2, n_out)) / np.sqrt(n_in // 2)
    X = rng.standard_normal((rows, n_in)) * 2.0
    layer = pkg.Layer.from_host(n_in, n_out, G, P, gamma, precision=64)
    ref = oracle.forward(G, P, X, gamma)
    _assert_bits(layer.forward(torch.from_numpy(X).cuda()).cpu().numpy(), ref)
    # fp32 I/O: the fp64 result rounded once
    Xf = X.astype(np.float32)
    ref32 = oracle.forward(G, P, Xf.astype(np.float64), gamma).astype(np.float32)
    Yf = layer.forward(torch.from_numpy(Xf).cuda()).cpu().numpy()
    assert np.array_equal(Yf.view(np.uint32), ref32.view(np.uint32))
    assert np.array_equal(layer.read_table(), P)


def test_exact_layer_refusals(torch, pkg):
    P = np.zeros((5, 5, 2, 4))
    layer = pkg.Layer.from_host(4, 4, 4, P, 1.0, precision=64)
    X = torch.zeros((3, 4), device="cuda")
    with pytest.raises(ValueError, match="plain forward only"):
        layer.forward_dests(X, [torch.zeros((3, 8), device="cuda").data_ptr()], 8, 4)
    with pytest.raises(ValueError, match="reference-precision"):
        layer.records(X, "in_kernel")
    with pytest.raises(ValueError, match="reference-precision"):
        pkg.Model.from_layers([layer])


def test_exact_staged_records_and_row_chunks(torch, pkg, oracle, monkeypatch):
    """Layers with several output tiles stage the fp64 cell records (one
    locate per (row, pair) instead of one per output tile); the staged path,
    its row chunks under a small scratch cap, and the fused kernel all give
    the reference's bits."""
    n_in, n_out, G, rows = 40, 96, 12, 5000
    rng = np.random.default_rng(11)
    P = rng.standard_normal((G + 1, G + 1, n_in // 2, n_out)) / np.sqrt(n_in // 2)
    X = rng.standard_normal((rows, n_in)) * 1.5
    layer = pkg.Layer.from_host(n_in, n_out, G, P, 1.0, precision=64)
    ref = oracle.forward(G, P, X, 1.0)
    Xd = torch.from_numpy(X).cuda()
    for env in ({}, {"LMKAN_B200_MAX_SCRATCH_MB": "1"}, {"LMKAN_B200_EXACT_STAGED": "0"}):
        for k in ("LMKAN_B200_MAX_SCRATCH_MB", "LMKAN_B200_EXACT_STAGED"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        _assert_bits(layer.forward(Xd).cpu().numpy(), ref)
