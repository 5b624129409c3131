"""BASELINE.json configs at their FULL sizes (the bench workloads), checked
through size-independent properties, with oracle parity on row subsets:

  * row independence (layer.hpp:118-132): the full-batch forward equals the
    forwards of arbitrary row splits, bitwise (batch sharding, configs 1-4);
  * output independence (layer.hpp:128-129): output slices reproduce columns
    bitwise (output sharding, config 5);
  * gamma linearity: gamma = 0.5 gives exactly half of gamma = 1 (the final
    multiply by a power of two is exact);
  * parity with the reference (|y - y_ref| <= 1e-5 max(1, |y_ref|)) on rows
    drawn from across the whole batch, and the production cell records of
    those rows bit-exact.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-5


def _sample_rows(n, k, seed):
    rng = np.random.default_rng(seed)
    idx = np.sort(rng.choice(n, size=k, replace=False))
    idx[0], idx[-1] = 0, n - 1  # both ends of the batch
    return idx


def _check_rows(oracle, layer, X, Y, rows, G):
    import pyoracle
    Xs = X[rows].double().cpu().numpy()
    ref = oracle.forward(G, layer.read_table(), Xs, 1.0)
    assert pyoracle.mixed_err(Y[rows].cpu().numpy(), ref).max() <= TOL
    r1, r2, _ = oracle.locate(G, Xs)
    i1, i2, _ = layer.records(X[rows].contiguous(), "k1" if layer.plan(len(rows))["mode"] != "narrow" else "in_kernel")
    assert np.array_equal(i1.cpu().numpy(), r1) and np.array_equal(i2.cpu().numpy(), r2)


def test_cfg2_full_batch(torch, pkg, oracle):
    """1024 -> 1024, G = 16, 65536 rows (the default bench workload)."""
    n_in, n_out, G, B = 1024, 1024, 16, 65536
    layer = pkg.Layer.random(n_in, n_out, G, seed=1000)
    X = torch.randn((B, n_in), generator=torch.Generator(device="cuda").manual_seed(1234), device="cuda")
    Y = layer.forward(X)
    assert torch.equal(Y, layer.forward(X))  # run to run
    cuts = [0, 1, 4097, 33333, 65535, B]
    assert torch.equal(torch.cat([layer.forward(X[a:b].contiguous()) for a, b in zip(cuts, cuts[1:])]), Y)
    half = pkg.Layer.random(n_in, n_out, G, seed=1000, gamma=0.5)
    assert torch.equal(half.forward(X), Y * 0.5)
    for ob, oe in [(0, 64), (64, 448), (448, 1024)]:
        sl = pkg.Layer.random(n_in, n_out, G, seed=1000, out_range=(ob, oe))
        assert torch.equal(sl.forward(X), Y[:, ob:oe])
    _check_rows(oracle, layer, X, Y, _sample_rows(B, 24, 1), G)


def test_cfg3_full_chain(torch, pkg, oracle):
    """Methane chain 12 -> 128 -> 128 -> 1, G = 28, 2^20 rows (graph-replayed model)."""
    import pyoracle
    G, B = 28, 1 << 20
    layers = [pkg.Layer.random(a, b, G, seed=1000 + i) for i, (a, b) in enumerate([(12, 128), (128, 128), (128, 1)])]
    model = pkg.Model.from_layers(layers)
    X = torch.randn((B, 12), generator=torch.Generator(device="cuda").manual_seed(7), device="cuda")
    Y = model.infer(X)
    cuts = [0, 12345, 700001, B]
    assert torch.equal(torch.cat([model.infer(X[a:b].contiguous()) for a, b in zip(cuts, cuts[1:])]), Y)
    # the chain equals the three layer forwards back to back, bitwise ...
    acts = [X]
    for lay in layers:
        acts.append(lay.forward(acts[-1]))
    assert torch.equal(acts[-1], Y)
    # ... and each layer meets the parity bar on its own (device) inputs
    rows = _sample_rows(B, 64, 3)
    for lay, a, y in zip(layers, acts[:-1], acts[1:]):
        ref = oracle.forward(G, lay.read_table(), a[rows].double().cpu().numpy(), 1.0)
        assert pyoracle.mixed_err(y[rows].cpu().numpy(), ref).max() <= TOL


def test_cfg4_full_conv(torch, pkg, oracle):
    """3x3 conv 144 -> 16, G = 16, 256 zero-padded 34x34x16 images (262144 patch rows)."""
    import pyoracle
    G = 16
    layer = pkg.Layer.random(144, 16, G, seed=1000)
    img = torch.randn((256, 34, 34, 16), generator=torch.Generator(device="cuda").manual_seed(3), device="cuda")
    img[:, 0] = 0
    img[:, -1] = 0
    img[:, :, 0] = 0
    img[:, :, -1] = 0
    Y = layer.conv_forward(img, 3, 1)
    parts = [layer.conv_forward(img[a:b].contiguous(), 3, 1) for a, b in [(0, 1), (1, 100), (100, 256)]]
    assert torch.equal(torch.cat(parts), Y)
    # oracle on a few images' patch rows (unfold_conv column order (dy*3 + dx)*16 + ch)
    sel = [0, 131, 255]
    im = img[sel].cpu().numpy()
    cols = [im[:, dy:dy + 32, dx:dx + 32, :] for dy in range(3) for dx in range(3)]
    patches = np.concatenate(cols, axis=-1).reshape(-1, 144).astype(np.float64)
    ref = oracle.forward(G, layer.read_table(), patches, 1.0)
    assert pyoracle.mixed_err(Y[sel].reshape(-1, 16).cpu().numpy(), ref).max() <= TOL
