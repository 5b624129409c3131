"""GPU parity tests: the sm_100a path through the C-ABI vs the oracle.

Oracle = the reference's own lmkan_forward / row_preambles compiled from
/root/reference (oracle/_ref) when present, else the C restatement (oracle/).
Same inputs for both: fp32 X and fp32 P, widened exactly to double for the
oracle. Bars:
  * cell indices (i1, i2) bit-exact; weights == fp32(reference fp64 weight);
  * outputs |y - y_ref| <= 1e-5 * max(1, |y_ref|), the reference's own
    normalization (test_layer.cpp:96-97).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-5


@pytest.fixture(scope="module")
def torch():
    import torch as t
    return t


@pytest.fixture(scope="module")
def pkg():
    import paper_2509_07103_b200 as p
    return p


def _mixed(y, ref):
    import pyoracle
    return pyoracle.mixed_err(y, ref)


def _inputs(torch, n_in, n_out, G, rows, seed, xscale=1.0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    P = torch.randn((G + 1, G + 1, n_in // 2, n_out), generator=g, dtype=torch.float32) / np.sqrt(n_in // 2)
    X = torch.randn((rows, n_in), generator=g, dtype=torch.float32) * xscale
    return P.numpy(), X.numpy()


def _special_rows(n_in, G, pkg):
    """Rows built from the reference's edge cases: thresholds +-1 ulp, +-0,
    tiny negatives (exp(-|x|) rounds to 1), huge, +-inf, NaN."""
    t64, t32 = pkg.thresholds(G)
    vals = [0.0, -0.0, 1e-45, -1e-45, -1e-30, 1e-30, -5e-17, 5e-17, 3e38, -3e38, np.inf, -np.inf, np.nan,
            100.0, -100.0]
    for t in t32:
        vals += [np.nextafter(t, -np.inf, dtype=np.float32), t, np.nextafter(t, np.inf, dtype=np.float32)]
    vals = np.array(vals, np.float32)
    reps = int(np.ceil(vals.size * 2 / n_in)) + 1
    rng = np.random.default_rng(G)
    out = np.concatenate([rng.permutation(vals) for _ in range(reps * n_in // vals.size + 2)])
    return out[: reps * n_in].reshape(reps, n_in)


SHAPES = [  # (n_in, n_out, G, rows) — BASELINE.json configs, row subsets where the oracle is slow
    (64, 64, 8, 1024),      # cfg1
    (1024, 1024, 16, 300),  # cfg2 (row subset)
    (12, 128, 28, 4096),    # cfg3 layer 1
    (128, 128, 28, 2048),   # cfg3 layer 2
    (128, 1, 28, 4096),     # cfg3 head
    (144, 16, 16, 4096),    # cfg4 stage 1
    (288, 32, 16, 2048),    # cfg4 stage 2
    (576, 64, 16, 1024),    # cfg4 stage 3
]


@pytest.mark.parametrize("n_in,n_out,G,rows", SHAPES)
def test_locate_bit_exact(torch, pkg, oracle, n_in, n_out, G, rows):
    P, X = _inputs(torch, n_in, n_out, G, rows, seed=n_in + G)
    X = np.concatenate([X, _special_rows(n_in, G, pkg)])
    layer = pkg.Layer.from_host(n_in, n_out, G, P.astype(np.float64), 1.0)
    i1, i2, w = layer.locate(torch.from_numpy(X).cuda())
    r1, r2, rw = oracle.locate(G, X.astype(np.float64))
    assert np.array_equal(i1.cpu().numpy(), r1)
    assert np.array_equal(i2.cpu().numpy(), r2)
    np.testing.assert_array_equal(w.cpu().numpy(), rw.astype(np.float32))


@pytest.mark.parametrize("G", [3, 4, 5, 8, 12, 13, 16, 28, 32, 40, 64, 100, 255])
def test_locate_f64_near_thresholds(torch, pkg, oracle, G):
    """Double inputs that are not fp32-representable, packed around every
    threshold: the f64 path compares against the fp64 thresholds."""
    t64, _ = pkg.thresholds(G)
    xs = []
    for t in t64:
        x = t
        for _ in range(40):
            x = np.nextafter(x, -np.inf)
        for _ in range(80):
            xs.append(x)
            x = np.nextafter(x, np.inf)
    xs += [0.0, -0.0, -1e-300, 1e-300, -2.0 ** -54, -2.0 ** -53, np.inf, -np.inf, np.nan, 1e308, -1e308]
    xs = np.array(xs)
    if xs.size % 2:
        xs = np.append(xs, 0.25)
    X = xs.reshape(-1, 2)
    layer = pkg.Layer.random(2, 4, G, seed=1)
    i1, i2, w = layer.locate(torch.from_numpy(X).cuda())
    r1, r2, rw = oracle.locate(G, X)
    assert np.array_equal(i1.cpu().numpy(), r1)
    assert np.array_equal(i2.cpu().numpy(), r2)
    np.testing.assert_array_equal(w.cpu().numpy(), rw.astype(np.float32))


@pytest.mark.parametrize("n_in,n_out,G,rows", SHAPES)
def test_forward_parity(torch, pkg, oracle, n_in, n_out, G, rows):
    P, X = _inputs(torch, n_in, n_out, G, rows, seed=3 * n_in + G)
    layer = pkg.Layer.from_host(n_in, n_out, G, P.astype(np.float64), 1.0)
    Y = layer.forward(torch.from_numpy(X).cuda()).cpu().numpy()
    ref = oracle.forward(G, P.astype(np.float64), X.astype(np.float64), 1.0)
    err = _mixed(Y, ref)
    assert err.max() <= TOL, f"max mixed err {err.max():.3e}"


@pytest.mark.parametrize("n_in,n_out,G,rows,gamma", [
    (2, 1, 5, 64, 1.0), (6, 5, 3, 64, 0.8), (6, 5, 12, 64, 0.8), (8, 3, 4, 33, 0.6), (8, 6, 12, 33, 0.9),
    (4, 3, 4, 16, 0.0), (10, 7, 64, 130, 1.0), (30, 100, 9, 777, 1.3), (16, 20, 6, 1, 1.0),
    (64, 200, 8, 5000, 1.0), (256, 48, 20, 3001, 0.5),
    (10, 7, 100, 130, 1.0), (6, 5, 255, 50, 0.7),  # large grids: sheets read from L2 (global mode)
])
def test_forward_small_and_ragged(torch, pkg, oracle, n_in, n_out, G, rows, gamma):
    P, X = _inputs(torch, n_in, n_out, G, rows, seed=n_in * 7 + n_out + G, xscale=1.5)
    layer = pkg.Layer.from_host(n_in, n_out, G, P.astype(np.float64), gamma)
    Y = layer.forward(torch.from_numpy(X).cuda()).cpu().numpy()
    ref = oracle.forward(G, P.astype(np.float64), X.astype(np.float64), gamma)
    assert _mixed(Y, ref).max() <= TOL


def test_forward_nonfinite_inputs(torch, pkg, oracle):
    """+-inf / NaN inputs propagate like the reference: same NaN and +-inf
    positions, finite outputs within tolerance. (|x| is kept where the fp64
    weights stay inside fp32 range; beyond that fp32 outputs cannot represent
    the reference's finite huge values.)"""
    n_in, n_out, G = 32, 16, 8
    P, _ = _inputs(torch, n_in, n_out, G, 1, seed=5)
    X = _special_rows(n_in, G, pkg)
    X[np.isfinite(X) & (np.abs(X) > 1e4)] = 1e4
    finite_rows = X.copy()
    finite_rows[~np.isfinite(finite_rows)] = 0.5
    # |x| up to 100 (edge cells extrapolate with weights ~x^2/h^2; beyond that
    # fp32 cancellation between the huge edge weights exceeds 1e-5 relative
    # even though the fp64 reference stays exact-ish)
    finite_rows = np.clip(finite_rows, -100, 100)
    X = np.concatenate([X, finite_rows])
    layer = pkg.Layer.from_host(n_in, n_out, G, P.astype(np.float64), 1.0)
    Y = layer.forward(torch.from_numpy(X).cuda()).cpu().numpy().astype(np.float64)
    ref = oracle.forward(G, P.astype(np.float64), X.astype(np.float64), 1.0)
    assert np.array_equal(np.isnan(Y), np.isnan(ref))
    assert np.array_equal(np.isposinf(Y), np.isposinf(ref))
    assert np.array_equal(np.isneginf(Y), np.isneginf(ref))
    fin = np.isfinite(ref)
    assert fin.sum() >= X.shape[0] // 2 * n_out
    assert _mixed(Y[fin], ref[fin]).max() <= TOL


def test_forward_deterministic_and_shard_invariant(torch, pkg):
    n_in, n_out, G, rows = 256, 192, 16, 5000
    P, X = _inputs(torch, n_in, n_out, G, rows, seed=11)
    layer = pkg.Layer.from_host(n_in, n_out, G, P.astype(np.float64), 1.0)
    Xd = torch.from_numpy(X).cuda()
    Y1 = layer.forward(Xd)
    Y2 = layer.forward(Xd)
    assert torch.equal(Y1, Y2)
    # batch sharding (configs 1-4): any row split gives bitwise-identical rows
    parts = [layer.forward(Xd[a:b].contiguous()) for a, b in [(0, 1000), (1000, 1001), (1001, rows)]]
    assert torch.equal(torch.cat(parts), Y1)
    # output sharding (config 5): output-sliced layers reproduce columns bitwise
    Pd = torch.from_numpy(P).cuda()
    for ob, oe in [(0, 64), (64, 130), (130, 192)]:
        sl = pkg.Layer.from_device(n_in, n_out, G, Pd, 1.0, out_range=(ob, oe))
        assert torch.equal(sl.forward(Xd), Y1[:, ob:oe])


def test_table_roundtrip(torch, pkg):
    n_in, n_out, G = 12, 40, 5
    P, _ = _inputs(torch, n_in, n_out, G, 1, seed=2)
    layer = pkg.Layer.from_host(n_in, n_out, G, P.astype(np.float64), 1.0)
    np.testing.assert_array_equal(layer.read_table(), P.astype(np.float64))
    np.testing.assert_array_equal(layer.read_table(2, 5), P[:, :, 2:5].astype(np.float64))
    sl = pkg.Layer.from_device(n_in, n_out, G, torch.from_numpy(P).cuda(), 1.0, out_range=(7, 33))
    np.testing.assert_array_equal(sl.read_table(), P[..., 7:33].astype(np.float64))


def test_random_table_layer_matches_oracle(torch, pkg, oracle):
    n_in, n_out, G, rows = 64, 96, 8, 700
    layer = pkg.Layer.random(n_in, n_out, G, seed=99)
    P = layer.read_table()
    assert abs(P.std() * np.sqrt(n_in // 2) - 1.0) < 0.05
    _, X = _inputs(torch, n_in, n_out, G, rows, seed=4)
    Y = layer.forward(torch.from_numpy(X).cuda()).cpu().numpy()
    ref = oracle.forward(G, P, X.astype(np.float64), 1.0)
    assert _mixed(Y, ref).max() <= TOL


def test_host_paths(torch, pkg, oracle):
    """Drop-in host entry points (lmkan_forward semantics on host memory)."""
    n_in, n_out, G, rows = 48, 40, 8, 3000
    rng = np.random.default_rng(1)
    P = rng.normal(size=(G + 1, G + 1, n_in // 2, n_out)) / np.sqrt(n_in // 2)  # full fp64 table
    X = rng.normal(size=(rows, n_in))  # fp64, not fp32-representable
    lay = pkg.init_layer(n_in, n_out, G, seed=5)
    lay.P = P
    lay.gamma = 0.7
    Y = pkg.lmkan_forward(lay, X)
    ref = oracle.forward(G, P, X, 0.7)
    assert _mixed(Y, ref).max() <= TOL
    # in-place table edit is never served stale
    lay.P[0, 0, 0, 0] += 5.0
    Y2 = pkg.lmkan_forward(lay, X)
    ref2 = oracle.forward(G, lay.P, X, 0.7)
    assert _mixed(Y2, ref2).max() <= TOL
    # fp32 host path
    layer = lay.prepared()
    Xf = X.astype(np.float32)
    Yf = layer.forward_host(Xf)
    reff = oracle.forward(G, P.astype(np.float32).astype(np.float64) + 0.0, Xf.astype(np.float64), 0.7)
    reff = oracle.forward(G, layer.read_table(), Xf.astype(np.float64), 0.7)
    assert _mixed(Yf, reff).max() <= TOL
    with pytest.raises(ValueError, match="expected width 48, got 50"):
        pkg.lmkan_forward(lay, np.zeros((3, 50)))


def test_init_layer_forward_zero_gamma(torch, pkg):
    lay = pkg.init_layer(4, 3, 4, 123)
    assert lay.gamma == 0.0
    Y = pkg.lmkan_forward(lay, np.random.default_rng(0).normal(size=(16, 4)))
    assert (Y == 0).all()


def test_f64_device_path(torch, pkg, oracle):
    n_in, n_out, G, rows = 40, 24, 13, 999
    layer = pkg.Layer.random(n_in, n_out, G, seed=3)
    X = np.random.default_rng(2).normal(size=(rows, n_in)) * 2
    Y = layer.forward(torch.from_numpy(X).cuda()).cpu().numpy()
    ref = oracle.forward(G, layer.read_table(), X, 1.0)
    assert _mixed(Y, ref).max() <= TOL


@pytest.mark.parametrize("n_in,n_out,G,rows", [(128, 128, 28, 30000),   # staged, 1024-row tiles, GOFF
                                               (144, 16, 16, 20000),     # fused, DUP table
                                               (256, 64, 16, 20000)])    # staged, V = 4 lane runs
def test_f64_io_matches_f32_io_bitwise(torch, pkg, oracle, n_in, n_out, G, rows):
    """fp64 I/O runs the same fp32 gathers: on fp32-representable inputs the
    cells (fp64 vs fp32 thresholds) and {alpha, gamma} agree, so Y is the fp32
    path's Y widened, bit for bit, in every kernel family; and it meets the
    parity bar."""
    layer = pkg.Layer.random(n_in, n_out, G, seed=n_in + G)
    X32 = torch.randn((rows, n_in), device="cuda") * 1.3
    Y32 = layer.forward(X32)
    Y64 = layer.forward(X32.double())
    assert Y64.dtype == torch.float64
    assert torch.equal(Y64, Y32.double())
    ref = oracle.forward(G, layer.read_table(), X32[:300].double().cpu().numpy(), 1.0)
    assert _mixed(Y64[:300].cpu().numpy(), ref).max() <= TOL


VARIANTS = [("fused", "1", "16"), ("fused", "2", "8"), ("fused", "3", "4"), ("staged", "1", "16"),
            ("staged", "2", "16"), ("staged", "3", "8"), ("staged", "4", "4"), ("global", "1", "4"),
            # OT = 64 runs two float4 runs per lane: rows per thread 8 / 4 / 2
            ("staged", "1", "2"), ("fused", "2", "2"), ("global", "1", "2")]


@pytest.mark.parametrize("G", [8, 28, 32])
def test_kernel_variants_parity_and_bitwise_agreement(torch, pkg, oracle, monkeypatch, G):
    """Every kernel variant (fused / staged / global-sheet, 1-4 i1-slabs, row
    tiles) meets the parity bar AND agrees bitwise with every other variant:
    the per-(row, output) summation order does not depend on the variant."""
    n_in, n_out, rows = 40, 72, 1300
    P, X = _inputs(torch, n_in, n_out, G, rows, seed=G + 100, xscale=1.3)
    Xd = torch.from_numpy(X).cuda()
    ref = oracle.forward(G, P.astype(np.float64), X.astype(np.float64), 1.0)
    outs = []
    for ot in ("16", "32", "64"):
        monkeypatch.setenv("LMKAN_B200_OT", ot)
        layer = pkg.Layer.from_host(n_in, n_out, G, P.astype(np.float64), 1.0)
        for mode, slabs, rt in VARIANTS:
            monkeypatch.setenv("LMKAN_B200_MODE", mode)
            monkeypatch.setenv("LMKAN_B200_SLABS", slabs)
            monkeypatch.setenv("LMKAN_B200_RT", rt)
            try:
                plan = layer.plan(rows)
            except ValueError:
                continue  # this variant does not fit shared memory at this G / OT
            assert plan["mode"] == mode and str(plan["slabs"]) == slabs and str(plan["rows_per_thread"]) == rt
            Y = layer.forward(Xd)
            assert _mixed(Y.cpu().numpy(), ref).max() <= TOL, (ot, mode, slabs, rt)
            outs.append(((ot, mode, slabs, rt), Y))
        for k in ("LMKAN_B200_MODE", "LMKAN_B200_SLABS", "LMKAN_B200_RT"):
            monkeypatch.delenv(k)
    assert len(outs) >= 8
    base = outs[0][1]
    for name, Y in outs[1:]:
        assert torch.equal(Y, base), name


@pytest.mark.parametrize("ot", ["64", "16"])
def test_small_batch_warps_per_cta(torch, pkg, oracle, monkeypatch, ot):
    """Small batches run CTAs of 8/4/2/1 warps (4 float4s per thread) so the grid spans at
    least half the GPU; every warps-per-CTA choice meets the parity bar and is bitwise equal
    to the 16-warp launch (the per-row summation order does not change)."""
    n_in, n_out, G, rows = 64, 64, 8, 1024  # config 1
    P, X = _inputs(torch, n_in, n_out, G, rows, seed=77)
    Xd = torch.from_numpy(X).cuda()
    ref = oracle.forward(G, P.astype(np.float64), X.astype(np.float64), 1.0)
    monkeypatch.setenv("LMKAN_B200_OT", ot)
    layer = pkg.Layer.from_host(n_in, n_out, G, P.astype(np.float64), 1.0)
    auto = layer.plan(rows)
    ctas = -(-rows // auto["rows_per_cta"]) * -(-n_out // auto["out_tile"])
    assert auto["warps_per_cta"] < 16 and (2 * ctas >= 148 or auto["warps_per_cta"] == 1), auto
    outs = []
    small_rt = str(4 // auto["lane_vectors"])  # the small-batch register tile: 4 float4s per thread
    for mode in ("fused", "staged"):
        monkeypatch.setenv("LMKAN_B200_MODE", mode)
        for nw in ("16", "8", "4", "2", "1"):
            monkeypatch.setenv("LMKAN_B200_NW", nw)
            monkeypatch.setenv("LMKAN_B200_RT", small_rt)
            plan = layer.plan(rows)
            assert plan["warps_per_cta"] == int(nw) and plan["mode"] == mode, plan
            Y = layer.forward(Xd)
            assert _mixed(Y.cpu().numpy(), ref).max() <= TOL, (mode, nw)
            outs.append(((mode, nw), Y))
    for name, Y in outs[1:]:
        assert torch.equal(Y, outs[0][1]), name


def test_staged_row_chunking_bitwise(torch, pkg, monkeypatch):
    """Batches whose cell-record scratch exceeds the cap run in row chunks;
    results are bitwise identical to the unchunked launch."""
    n_in, n_out, G, rows = 256, 256, 16, 9000
    layer = pkg.Layer.random(n_in, n_out, G, seed=8)
    X = torch.randn((rows, n_in), device="cuda")
    monkeypatch.setenv("LMKAN_B200_MODE", "staged")
    Y1 = layer.forward(X)
    monkeypatch.setenv("LMKAN_B200_MAX_SCRATCH_MB", "2")  # 2 MB -> ~ 1.6k-row chunks
    Y2 = layer.forward(X)
    assert torch.equal(Y1, Y2)


def test_cfg5_shape_output_slice(torch, pkg, oracle):
    """Config-5 geometry (8192 -> 8192, G = 32, 4096 pairs per output): an
    output-sharded slice of the device-generated table, checked against the
    oracle on a row subset (the longest accumulation chain of any config)."""
    n_in, n_out, G, rows = 8192, 8192, 32, 48
    ob, oe = 4096, 4112
    layer = pkg.Layer.random(n_in, n_out, G, seed=55, out_range=(ob, oe))
    P = layer.read_table()
    X = torch.randn((rows, n_in), generator=torch.Generator().manual_seed(5)).float()
    Y = layer.forward(X.cuda()).cpu().numpy()
    ref = oracle.forward(G, P, X.double().numpy(), 1.0)
    assert _mixed(Y, ref).max() <= TOL


@pytest.mark.parametrize("n_in,n_out,G,rows", [(128, 1, 28, 3000), (64, 2, 16, 2000), (30, 3, 8, 999),
                                               (2, 4, 5, 100), (200, 1, 12, 513),
                                               # tables whose byte size is not a multiple of 16 (the bulk
                                               # copy moves the allocation's zeroed 16-B-rounded tail)
                                               (2, 1, 4, 77), (6, 1, 8, 300), (10, 2, 4, 129), (14, 2, 6, 64)])
def test_narrow_kernel(torch, pkg, oracle, monkeypatch, n_in, n_out, G, rows):
    """n_out <= 4 layers run the narrow kernel (whole table in shared memory,
    one row per lane); parity vs the oracle, bitwise vs the padded general path."""
    P, X = _inputs(torch, n_in, n_out, G, rows, seed=n_in + 7 * n_out)
    layer = pkg.Layer.from_host(n_in, n_out, G, P.astype(np.float64), 0.9)
    assert layer.plan(rows)["mode"] == "narrow"
    Xd = torch.from_numpy(X).cuda()
    Y = layer.forward(Xd).cpu().numpy()
    ref = oracle.forward(G, P.astype(np.float64), X.astype(np.float64), 0.9)
    assert _mixed(Y, ref).max() <= TOL
    assert np.array_equal(layer.forward(Xd).cpu().numpy(), Y)  # deterministic
    monkeypatch.setenv("LMKAN_B200_NARROW", "0")
    wide = pkg.Layer.from_host(n_in, n_out, G, P.astype(np.float64), 0.9)
    assert wide.plan(rows)["mode"] != "narrow"
    # same per-(row, output) arithmetic and pair order as the general kernel
    assert np.array_equal(wide.forward(Xd).cpu().numpy(), Y)


def _unfold(img, k, s):
    """unfold_conv (conv.hpp:39-60) restated in numpy: rows over (n, oy, ox),
    columns (dy*k + dx)*C + ch."""
    N, H, W, C = img.shape
    oh, ow = (H - k) // s + 1, (W - k) // s + 1
    cols = []
    for dy in range(k):
        for dx in range(k):
            cols.append(img[:, dy:dy + s * (oh - 1) + 1:s, dx:dx + s * (ow - 1) + 1:s, :])
    return np.concatenate(cols, axis=-1).reshape(N * oh * ow, k * k * C), oh, ow


@pytest.mark.parametrize("N,H,W,C,k,s,n_out,G", [
    (4, 10, 10, 16, 3, 1, 16, 16),   # CIFAR stage-1 geometry, small batch
    (2, 9, 9, 2, 3, 3, 7, 8),
    (3, 8, 8, 6, 2, 2, 40, 5),
    (2, 7, 9, 3, 2, 1, 10, 6),       # odd C: x pairs straddle taps
    (2, 6, 6, 4, 3, 1, 2, 12),       # narrow head (n_out <= 4)
    (3, 18, 18, 32, 3, 1, 32, 16),   # CIFAR stage-2 geometry (OT 32)
    (2, 10, 10, 64, 3, 1, 64, 16),   # CIFAR stage-3 geometry (OT 64)
    (2, 11, 13, 8, 3, 2, 24, 9),     # stride 2, non-square
])
def test_conv_implicit_im2col(torch, pkg, oracle, N, H, W, C, k, s, n_out, G):
    rng = np.random.default_rng(N * 100 + C)
    img = rng.standard_normal((N, H, W, C)).astype(np.float32)
    n_in = k * k * C
    P = (rng.standard_normal((G + 1, G + 1, n_in // 2, n_out)) / np.sqrt(n_in // 2)).astype(np.float32)
    layer = pkg.Layer.from_host(n_in, n_out, G, P.astype(np.float64), 1.0)
    Y = layer.conv_forward(torch.from_numpy(img).cuda(), k, s)
    patches, oh, ow = _unfold(img, k, s)
    assert Y.shape == (N, oh, ow, n_out)  # fold_output layout (conv.hpp:63-71)
    Yx = layer.forward(torch.from_numpy(np.ascontiguousarray(patches)).cuda())
    assert torch.equal(Y.reshape(-1, n_out), Yx)  # same rows, same kernel, same order
    ref = oracle.forward(G, P.astype(np.float64), patches.astype(np.float64), 1.0)
    assert _mixed(Y.reshape(-1, n_out).cpu().numpy(), ref).max() <= TOL
    # host entry (image chunks over two streams): same bits as the device call
    assert np.array_equal(layer.conv_forward_host(img, k, s), Y.cpu().numpy())


def test_conv_host_chunked_cfg4_shape(torch, pkg):
    """cfg4 geometry through the host conv entry (several image chunks) equals
    the single device launch bitwise."""
    rng = np.random.default_rng(4)
    img = rng.standard_normal((300, 34, 34, 16)).astype(np.float32)
    layer = pkg.Layer.random(144, 16, 16, seed=4)
    Yd = layer.conv_forward(torch.from_numpy(img).cuda(), 3, 1).cpu().numpy()
    assert np.array_equal(layer.conv_forward_host(img, 3, 1), Yd)


@pytest.mark.parametrize("N,H,W,C,n_out,G", [(40, 34, 34, 16, 16, 16), (20, 18, 18, 32, 32, 16),
                                             (10, 10, 10, 64, 64, 16), (6, 9, 9, 6, 20, 28)])
def test_conv_pixel_records_bitwise(torch, pkg, monkeypatch, N, H, W, C, n_out, G):
    """Records located once per image pixel (pixel_records_kernel, kModePixel)
    give the same output bits as the per-(row, pair) in-kernel locate."""
    rng = np.random.default_rng(C + N)
    img = torch.from_numpy(rng.standard_normal((N, H, W, C)).astype(np.float32) * 1.4).cuda()
    layer = pkg.Layer.random(9 * C, n_out, G, seed=C)
    Y = layer.conv_forward(img, 3, 1)
    monkeypatch.setenv("LMKAN_B200_PIXREC", "0")
    Y0 = layer.conv_forward(img, 3, 1)
    assert torch.equal(Y, Y0)


def test_conv_argument_errors(torch, pkg):
    layer = pkg.Layer.random(2 * 2 * 4, 8, 5)
    img = torch.zeros((1, 7, 7, 4), device="cuda")
    with pytest.raises(ValueError, match="divisible by the stride"):
        layer.conv_forward(img, 2, 2)
    with pytest.raises(ValueError, match="kernel larger than image"):
        layer.conv_forward(torch.zeros((1, 1, 1, 4), device="cuda"), 2, 1)
    with pytest.raises(ValueError, match="expected width 16, got 36"):
        layer.conv_forward(img, 3, 1)


@pytest.mark.parametrize("mode", ["fused", "staged"])
def test_balanced_row_tiles_bitwise(torch, pkg, oracle, monkeypatch, mode):
    """Row tiles shortened to whole warps so the grid fills the SMs (cfg4-like:
    128 CTAs of 2048 rows -> 147 of 1792): bitwise equal to the full-tile
    launch, and within the parity bar of the oracle on a row subset."""
    n_in, n_out, G, rows = 32, 16, 8, 250000
    rng = np.random.default_rng(12)
    P = (rng.standard_normal((G + 1, G + 1, n_in // 2, n_out)) / 4).astype(np.float32)
    layer = pkg.Layer.from_host(n_in, n_out, G, P.astype(np.float64), 1.0)
    X = torch.randn((rows, n_in), device="cuda")
    monkeypatch.setenv("LMKAN_B200_MODE", mode)
    outs = []
    for bal in ("0", "1"):
        monkeypatch.setenv("LMKAN_B200_BALANCE", bal)
        outs.append((layer.plan(rows), layer.forward(X)))
    (p_full, y_full), (p_bal, y_bal) = outs
    assert p_bal["rows_per_cta"] < p_full["rows_per_cta"], (p_full, p_bal)
    assert torch.equal(y_full, y_bal)
    ref = oracle.forward(G, P.astype(np.float64), X[:400].cpu().numpy().astype(np.float64), 1.0)
    assert _mixed(y_bal[:400].cpu().numpy(), ref).max() <= TOL


@pytest.mark.parametrize("n_in,n_out,G,force_ot", [(40, 16, 16, None), (30, 13, 8, None), (24, 40, 12, "16")])
def test_duplicated_node_tables_bitwise(torch, pkg, oracle, monkeypatch, n_in, n_out, G, force_ot):
    """OT = 16 layers store every node twice (conflict-free gathers): the
    table reads back as the reference P, and every mode / row tile gives the
    same bits as the plain table, within the parity bar of the oracle."""
    if force_ot:
        monkeypatch.setenv("LMKAN_B200_OT", force_ot)
    rows = 5000
    P, X = _inputs(torch, n_in, n_out, G, rows, seed=n_in + G)
    Xd = torch.from_numpy(X).cuda()
    ref = oracle.forward(G, P.astype(np.float64), X.astype(np.float64), 1.0)
    layers = {}
    for dup in ("0", "1"):
        monkeypatch.setenv("LMKAN_B200_DUP16", dup)
        layers[dup] = pkg.Layer.from_host(n_in, n_out, G, P.astype(np.float64), 1.0)
        r = pkg.Layer.random(n_in, n_out, G, seed=5)
        layers["rand" + dup] = r
    assert layers["1"].out_tile == 16 and layers["1"].table_bytes == 2 * layers["0"].table_bytes
    np.testing.assert_array_equal(layers["1"].read_table(), P.astype(np.float64))
    np.testing.assert_array_equal(layers["rand1"].read_table(), layers["rand0"].read_table())
    base = layers["0"].forward(Xd)
    lv = layers["1"].plan(rows)["lane_vectors"]  # 2: two 32-B runs per lane on duplicated-node tables
    for mode in ("fused", "staged"):
        monkeypatch.setenv("LMKAN_B200_MODE", mode)
        for rt in (str(16 // lv), str(8 // lv), str(4 // lv)):
            monkeypatch.setenv("LMKAN_B200_RT", rt)
            Y = layers["1"].forward(Xd)
            assert _mixed(Y.cpu().numpy(), ref).max() <= TOL, (mode, rt)
            assert torch.equal(Y, base), (mode, rt)
    monkeypatch.delenv("LMKAN_B200_RT")
    monkeypatch.delenv("LMKAN_B200_MODE")
    assert torch.equal(layers["rand1"].forward(Xd), layers["rand0"].forward(Xd))


@pytest.mark.parametrize("rows", [30000, 150000])  # balanced (shortened) tall tiles / full tiles
def test_global_offsets_tall_tile_bitwise(torch, pkg, oracle, monkeypatch, rows):
    """Staged layers whose ring only fits the taller row tile with the node
    offsets read from global memory (cfg3's 128->128 G=28 layer: 1024 rows per
    CTA instead of 512) give the same bits as the shorter tile, within the
    parity bar."""
    n_in, n_out, G = 128, 128, 28
    P, X = _inputs(torch, n_in, n_out, G, rows, seed=28)
    layer = pkg.Layer.from_host(n_in, n_out, G, P.astype(np.float64), 1.0)
    Xd = torch.from_numpy(X).cuda()
    outs = {}
    for goff in ("1", "0"):
        monkeypatch.setenv("LMKAN_B200_GOFF", goff)
        outs[goff] = (layer.plan(rows), layer.forward(Xd))
    assert outs["1"][0]["rows_per_thread"] == 2 * outs["0"][0]["rows_per_thread"], (outs["1"][0], outs["0"][0])
    assert outs["1"][0]["rows_per_cta"] > 512, outs["1"][0]
    assert torch.equal(outs["1"][1], outs["0"][1])
    sub = slice(0, 2000)
    ref = oracle.forward(G, P.astype(np.float64), X[sub].astype(np.float64), 1.0)
    assert _mixed(outs["1"][1][sub].cpu().numpy(), ref).max() <= TOL


def test_empty_batches(torch, pkg):
    """Zero rows (or zero images) are a no-op on every entry, like the
    reference's lmkan_forward on an empty Matrix (layer.hpp:111-118)."""
    layer = pkg.Layer.random(16, 8, 6, seed=1)
    Y = layer.forward(torch.empty((0, 16), device="cuda"))
    assert tuple(Y.shape) == (0, 8)
    for dt in (np.float32, np.float64):
        assert layer.forward_host(np.empty((0, 16), dt)).shape == (0, 8)
    assert pkg.lmkan_forward(pkg.init_layer(16, 8, 6, seed=1), np.empty((0, 16))).shape == (0, 8)
    conv = pkg.Layer.random(2 * 2 * 4, 8, 5, seed=2)
    assert tuple(conv.conv_forward(torch.zeros((0, 6, 6, 4), device="cuda"), 2, 1).shape) == (0, 5, 5, 8)
    assert conv.conv_forward_host(np.zeros((0, 6, 6, 4), np.float32), 2, 1).shape == (0, 5, 5, 8)
    m = pkg.Model.from_layers([pkg.Layer.random(12, 32, 8, seed=3), pkg.Layer.random(32, 2, 8, seed=4)])
    assert m.infer_host(np.empty((0, 12), np.float32)).shape == (0, 2)
    assert tuple(m.infer(torch.empty((0, 12), device="cuda")).shape) == (0, 2)


@pytest.mark.parametrize("taper", ["0", "1"])
def test_host_pipeline_multichunk_bitwise(torch, pkg, monkeypatch, taper):
    """The host entry points stream rows through the three-stage pipeline in
    several (optionally tapered) chunks; results equal the single device launch
    bitwise, for the layer, the model chain and odd chunk remainders."""
    monkeypatch.setenv("LMKAN_B200_HOST_TAPER", taper)
    monkeypatch.setenv("LMKAN_B200_HOST_CHUNKS", "7")
    layer = pkg.Layer.random(256, 96, 10, seed=21)
    rows = 123457
    X = torch.randn((rows, 256), device="cuda")
    Yd = layer.forward(X).cpu().numpy()
    Xh = X.cpu().numpy()
    assert np.array_equal(layer.forward_host(Xh), Yd)
    m = pkg.Model.from_layers([pkg.Layer.random(12, 64, 8, seed=3), pkg.Layer.random(64, 2, 8, seed=4)])
    Xm = torch.randn((300001, 12), device="cuda")
    assert np.array_equal(m.infer_host(Xm.cpu().numpy()), m.infer(Xm).cpu().numpy())


@pytest.mark.parametrize("n_in,n_out,G,rows,mode", [(64, 64, 8, 60000, "staged"), (64, 32, 8, 120000, "staged"),
                                                     (64, 64, 8, 60000, "fused"), (48, 32, 12, 120000, "fused")])
def test_balanced_tiles_lane_runs_bitwise(torch, pkg, oracle, monkeypatch, n_in, n_out, G, rows, mode):
    """Shortened (balanced) row tiles with several float4 runs per lane
    (OT = 64: V = 4, OT = 32: V = 2, bank-half interleave) give the same bits
    as the full tiles and meet the parity bar."""
    rng = np.random.default_rng(rows + n_out)
    P = (rng.standard_normal((G + 1, G + 1, n_in // 2, n_out)) / np.sqrt(n_in // 2)).astype(np.float32)
    monkeypatch.setenv("LMKAN_B200_OT", str(n_out))  # one n_out-wide tile: V = n_out / 16 runs per lane
    layer = pkg.Layer.from_host(n_in, n_out, G, P.astype(np.float64), 1.0)
    X = torch.randn((rows, n_in), device="cuda")
    monkeypatch.setenv("LMKAN_B200_MODE", mode)
    outs = []
    for bal in ("0", "1"):
        monkeypatch.setenv("LMKAN_B200_BALANCE", bal)
        outs.append((layer.plan(rows), layer.forward(X)))
    (p_full, y_full), (p_bal, y_bal) = outs
    assert p_bal["lane_vectors"] == n_out // 16 and p_bal["rows_per_cta"] < p_full["rows_per_cta"], (p_full, p_bal)
    assert torch.equal(y_full, y_bal)
    ref = oracle.forward(G, P.astype(np.float64), X[:300].double().cpu().numpy(), 1.0)
    assert _mixed(y_bal[:300].cpu().numpy(), ref).max() <= TOL


def test_output_slices_across_table_layouts_bitwise(torch, pkg):
    """Output slices of one layer land on different table layouts (64-wide
    tiles with 4 float4 runs per lane, 32-wide with 2, 16-wide duplicated-node
    tables); every slice equals the matching columns of the full layer, bit for
    bit, and its table reads back exactly."""
    n_in, n_out, G, rows = 40, 304, 12, 6000
    rng = np.random.default_rng(40)
    P = (rng.standard_normal((G + 1, G + 1, n_in // 2, n_out)) / np.sqrt(n_in // 2)).astype(np.float32)
    Pd = torch.from_numpy(P).cuda()
    X = torch.randn((rows, n_in), device="cuda")
    full = pkg.Layer.from_device(n_in, n_out, G, Pd, 1.0)
    Y = full.forward(X)
    widths = set()
    for ob, oe in [(0, 16), (16, 48), (48, 112), (112, 304), (100, 112)]:
        sl = pkg.Layer.from_device(n_in, n_out, G, Pd, 1.0, out_range=(ob, oe))
        widths.add(sl.out_tile)
        assert torch.equal(sl.forward(X), Y[:, ob:oe]), (ob, oe, sl.out_tile)
        np.testing.assert_array_equal(sl.read_table(), P[..., ob:oe].astype(np.float64))
    assert widths == {16, 32, 64}, widths


@pytest.mark.parametrize("x_pinned,y_pinned", [(False, False), (True, False), (False, True), (True, True)])
@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_host_staging_paths_bitwise(torch, pkg, monkeypatch, x_pinned, y_pinned, dtype):
    """Host entry points with pageable and/or pinned caller buffers: pageable
    ones are staged through pinned slots by the copy pool (non-temporal copies,
    fp64 Y crossing PCIe as fp32 and widened on the host). Every combination
    equals the device path bitwise, over several chunks with a ragged tail."""
    monkeypatch.setenv("LMKAN_B200_HOST_CHUNKS", "5")
    layer = pkg.Layer.random(96, 80, 12, seed=33)
    rows = 70001
    tdt = getattr(torch, dtype)
    Xd = (torch.randn((rows, 96), device="cuda", dtype=torch.float64) * 1.3).to(tdt)
    want = layer.forward(Xd).cpu().numpy()
    Xh = Xd.cpu().pin_memory() if x_pinned else Xd.cpu()
    Yh = torch.empty((rows, 80), dtype=tdt).pin_memory() if y_pinned else torch.empty((rows, 80), dtype=tdt)
    Yh.fill_(float("nan"))
    layer.forward_host_ptr(Xh.data_ptr(), Yh.data_ptr(), rows, np.dtype(dtype).type)
    assert np.array_equal(Yh.numpy(), want)
    assert np.array_equal(layer.forward_host(Xh.numpy()), want)


@pytest.mark.parametrize("n_in,n_out,G,rows,mode", [(64, 1024, 8, 5000, "staged"), (2304, 160, 4, 3000, "staged"),
                                                     (64, 200, 8, 40000, "fused")])
def test_cta_order_groups_bitwise(torch, pkg, oracle, monkeypatch, n_in, n_out, G, rows, mode):
    """The gather grid's CTA order (cta_tile, LMKAN_B200_CTA_GROUP) changes
    only which CTA runs which (row tile, output tile): every group size —
    including a last, partial group and the pair-block fold (1152 pairs), which
    re-derives its tile from the special registers — gives the same bits."""
    rng = np.random.default_rng(n_in + n_out)
    P = (rng.standard_normal((G + 1, G + 1, n_in // 2, n_out)) / np.sqrt(n_in // 2)).astype(np.float32)
    layer = pkg.Layer.from_host(n_in, n_out, G, P.astype(np.float64), 1.0)
    X = torch.randn((rows, n_in), device="cuda")
    monkeypatch.setenv("LMKAN_B200_MODE", mode)
    outs = []
    for g in ("1", "3", "4", "64"):
        monkeypatch.setenv("LMKAN_B200_CTA_GROUP", g)
        p = layer.plan(rows)
        assert p["mode"] == mode and p["cta_group"] == min(int(g), -(-n_out // p["out_tile"])), p
        outs.append(layer.forward(X))
    for y in outs[1:]:
        assert torch.equal(y, outs[0])
    ref = oracle.forward(G, P.astype(np.float64), X[:200].double().cpu().numpy(), 1.0)
    assert _mixed(outs[0][:200].cpu().numpy(), ref).max() <= TOL


@pytest.mark.parametrize("n_in,n_out,G,rows,ot,mode", [
    (576, 64, 16, 16384, 16, "staged"),    # conv stage 3: four OT = 16 tiles, cells staged once
    (128, 64, 28, 65536, 16, "staged"),
    (64, 64, 8, 1024, 64, "staged"),       # config 1: G < 12 keeps the one wide tile
    (288, 32, 16, 65536, 32, "fused"),     # two tiles at most: the single fused tile
    (1024, 1024, 16, 65536, 64, "staged"),  # config 2
    (128, 128, 28, 65536, 32, "staged"),   # config 3 layer 2
])
def test_output_tile_choice(torch, pkg, oracle, n_in, n_out, G, rows, ot, mode):
    """choose_out_tile: with G >= 12 the widest tile that still gives >= 3
    output tiles (the planner then stages the cells), else the widest that
    double-buffers; the chosen layout meets the parity bar."""
    layer = pkg.Layer.random(n_in, n_out, G, seed=3)
    p = layer.plan(rows)
    assert (layer.out_tile, p["mode"]) == (ot, mode), p
    X = torch.randn((min(rows, 4096), n_in), device="cuda")
    ref = oracle.forward(G, layer.read_table(), X[:64].double().cpu().numpy(), 1.0)
    assert _mixed(layer.forward(X)[:64].cpu().numpy(), ref).max() <= TOL


def test_conv_plan_pixel_ring(torch, pkg):
    """lmkan_b200_conv_plan: pixel records for even channel counts in the fused
    mode; the sheet ring is capped only when the CTA's pixel records then fit
    the L1 it leaves (conv stage 2), not when they fit no L1 (config 4)."""
    s2 = pkg.Layer.random(288, 32, 16, seed=1).conv_plan(256, 18, 18, 32, 3, 1)
    c4 = pkg.Layer.random(144, 16, 16, seed=1).conv_plan(256, 34, 34, 16, 3, 1)
    assert s2["pixel_records"] and c4["pixel_records"], (s2, c4)
    assert s2["nbuf"] == 2 and c4["nbuf"] >= 4, (s2, c4)
    with pytest.raises(ValueError):
        pkg.Layer.random(144, 16, 16, seed=1).conv_plan(2, 2, 2, 16, 3, 1)  # kernel larger than the image
