"""The PRODUCTION cell index is bit-exact (north_star: "cell indices bit-exact").

The kernels that produce Y locate cells with cell_index_fast (an fp32 sigma
estimate accepted only when bracketed by the exact thresholds, else a binary
search; csrc/locate.cuh). These tests read back what those kernels actually
produce, through lmkan_b200_records_*:
  * "k1"        K1 records4_kernel's output, decoded from the packed slab/node
                offsets and {alpha, gamma} rings exactly where K2 reads them;
  * "k1_smem"   the shared-memory-tile K1 (records_kernel);
  * "in_kernel" the fused / global / narrow kernels' in-kernel locate;
and compare them with the reference's row_preambles (layer.hpp:96-101, via
oracle/_ref): (i1, i2) bit for bit, and {alpha, gamma} bit for bit against
fp32((points[i+1] - x) * (1 / (points[i+1] - points[i]))) in fp64, the value the
weights are formed from.
"""
import numpy as np
import pytest

from test_parity_gpu import SHAPES, _inputs, _special_rows

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t
    return t


@pytest.fixture(scope="module")
def pkg():
    import paper_2509_07103_b200 as p
    return p


def _expected_ag(pkg, G, X, i1, i2):
    pts = pkg.build_grid(G).points
    invh = 1.0 / (pts[1:] - pts[:-1])
    X = X.astype(np.float64)
    with np.errstate(invalid="ignore", over="ignore"):
        a = ((pts[i1 + 1] - X[:, 0::2]) * invh[i1]).astype(np.float32)
        g = ((pts[i2 + 1] - X[:, 1::2]) * invh[i2]).astype(np.float32)
    return np.stack([a, g], axis=-1)


def _check(pkg, oracle, layer, X_np, Xd, variants):
    r1, r2, _ = oracle.locate(layer.G, X_np.astype(np.float64))
    want_ag = _expected_ag(pkg, layer.G, X_np, r1, r2)
    for v in variants:
        i1, i2, ag = layer.records(Xd, v)
        i1, i2, ag = i1.cpu().numpy(), i2.cpu().numpy(), ag.cpu().numpy()
        bad = np.argwhere((i1 != r1) | (i2 != r2))
        assert bad.size == 0, f"{v}: {len(bad)} cell mismatches, first (row, pair) {bad[0]}: " \
                              f"x={X_np[bad[0][0], 2 * bad[0][1]:2 * bad[0][1] + 2]}"
        np.testing.assert_array_equal(ag, want_ag, err_msg=v)


def _variants(layer, rows):
    return ["in_kernel"] if layer.plan(rows)["mode"] == "narrow" else ["k1", "k1_smem", "in_kernel"]


@pytest.mark.parametrize("n_in,n_out,G,rows", SHAPES)
def test_production_records_bit_exact(torch, pkg, oracle, n_in, n_out, G, rows):
    P, X = _inputs(torch, n_in, n_out, G, rows, seed=11 * n_in + G)
    X = np.concatenate([X, _special_rows(n_in, G, pkg)])
    layer = pkg.Layer.from_host(n_in, n_out, G, P.astype(np.float64), 1.0)
    Xd = torch.from_numpy(X).cuda()
    _check(pkg, oracle, layer, X, Xd, _variants(layer, X.shape[0]))
    # the same rows as fp64 I/O (cells against the fp64 thresholds)
    _check(pkg, oracle, layer, X.astype(np.float64), Xd.double(), _variants(layer, X.shape[0]))


def test_production_records_cfg5_geometry(torch, pkg, oracle):
    """8192 -> 8192, G = 32 (an output slice: records do not depend on n_out)."""
    n_in, G = 8192, 32
    layer = pkg.Layer.random(n_in, 8192, G, seed=3, out_range=(0, 16))
    X = np.concatenate([np.random.default_rng(5).standard_normal((40, n_in)).astype(np.float32),
                        _special_rows(n_in, G, pkg)])
    _check(pkg, oracle, layer, X, torch.from_numpy(X).cuda(), ["k1", "k1_smem", "in_kernel"])


@pytest.mark.parametrize("G", [3, 4, 5, 8, 12, 13, 16, 28, 32, 40, 64, 100, 255])
def test_production_records_f64_near_thresholds(torch, pkg, oracle, G):
    """Doubles packed +-40 ulps around every fp64 threshold (not fp32
    representable), plus +-0, tiny negatives, +-inf, NaN, huge values."""
    t64, t32 = pkg.thresholds(G)
    xs = []
    for t in t64:
        x = t
        for _ in range(40):
            x = np.nextafter(x, -np.inf)
        for _ in range(80):
            xs.append(x)
            x = np.nextafter(x, np.inf)
    xs += [0.0, -0.0, -1e-300, 1e-300, -2.0 ** -54, -2.0 ** -53, np.inf, -np.inf, np.nan, 1e308, -1e308]
    X = np.array(xs + [0.25] * (len(xs) % 2)).reshape(-1, 2)
    layer = pkg.Layer.random(2, 16, G, seed=1)
    # large grids run in global mode only (sheets from L2): no K1 records there
    variants = ["in_kernel"] if layer.plan(X.shape[0])["mode"] == "global" else ["k1", "k1_smem", "in_kernel"]
    _check(pkg, oracle, layer, X, torch.from_numpy(X).cuda(), variants)
    # fp32 inputs +-8 ulps around every fp32 threshold
    xs = []
    for t in t32:
        x = np.float32(t)
        for _ in range(8):
            x = np.nextafter(x, np.float32(-np.inf))
        for _ in range(16):
            xs.append(x)
            x = np.nextafter(x, np.float32(np.inf))
    X = np.array(xs + [np.float32(0.5)] * (len(xs) % 2), np.float32).reshape(-1, 2)
    _check(pkg, oracle, layer, X, torch.from_numpy(X).cuda(), variants)


@pytest.mark.parametrize("env,n_in,n_out,G,rows", [
    ({"LMKAN_B200_SLABS": "2"}, 128, 128, 28, 3000),   # slabbed sheets: slab bits in the packed offset
    ({"LMKAN_B200_SLABS": "3"}, 40, 64, 40, 777),
    ({}, 64, 64, 8, 60000),                              # balanced (shortened) row tiles
    ({"LMKAN_B200_RT": "4"}, 64, 32, 8, 5000),          # V = 2 lane runs, small tiles
    ({}, 128, 128, 28, 150000),                          # tall tiles, global node offsets (GOFF)
    ({}, 40, 16, 16, 20000),                             # duplicated-node (DUP) table: node stride 2 OT
])
def test_production_records_plan_variants(torch, pkg, oracle, monkeypatch, env, n_in, n_out, G, rows):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    layer = pkg.Layer.random(n_in, n_out, G, seed=n_in + G)
    X = np.random.default_rng(G).standard_normal((rows, n_in)).astype(np.float32) * 1.7
    sp = _special_rows(n_in, G, pkg)
    X[:len(sp)] = sp
    _check(pkg, oracle, layer, X, torch.from_numpy(X).cuda(), ["k1", "k1_smem", "in_kernel"])


def test_records_argument_errors(torch, pkg):
    narrow = pkg.Layer.random(8, 1, 8)
    X = torch.zeros((4, 8), device="cuda")
    with pytest.raises(ValueError):
        narrow.records(X, "k1")
    narrow.records(X, "in_kernel")
