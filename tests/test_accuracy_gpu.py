"""Accumulation accuracy at the longest pair chain (config 5: 8192 -> 8192, G = 32,
4096 pairs per output).

Each output is a sum over 4096 pairs (layer.hpp:128-129), accumulated in fp32
on the device. Layers with more than 1024 pairs sum in blocks of 256 pairs and
add the block sums in order (fwd_fused_kernel's pair-block summation), which
shrinks the rounding error ~4x. This scan checks >= 1e6 outputs of the config-5
geometry against the reference's fp64 lmkan_forward (oracle/_ref) and asserts
the 1e-5 bar (|y - y_ref| <= 1e-5 max(1, |y_ref|), test_layer.cpp:96-97) holds
with a margin of at least 1.5x.
"""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-5


def _scan(torch, pkg, oracle_ref, layer, P, n_in, rows, chunk, seed):
    import pyoracle
    G = layer.G
    ref_layer = pyoracle.RefLayer(oracle_ref, n_in, layer.n_out, G, P, 1.0) if oracle_ref is not None else None
    g = torch.Generator(device="cpu").manual_seed(seed)
    worst, n = 0.0, 0
    try:
        for r0 in range(0, rows, chunk):
            X = torch.randn((min(chunk, rows - r0), n_in), generator=g, dtype=torch.float32)
            Y = layer.forward(X.cuda()).cpu().numpy()
            Xd = X.double().numpy()
            ref = ref_layer.forward(Xd, 0) if ref_layer is not None else pyoracle.Port().forward(
                G, P, Xd, 1.0, threads=os.cpu_count() or 1)
            worst = max(worst, float(pyoracle.mixed_err(Y, ref).max()))
            n += Y.size
    finally:
        if ref_layer is not None:
            ref_layer.close()
    return worst, n


def test_cfg5_accumulation_margin(torch, pkg, monkeypatch):
    import pyoracle
    try:
        ref = pyoracle.Ref()
    except (FileNotFoundError, OSError):
        ref = None
    n_in, n_out, G = 8192, 8192, 32
    ob, oe = 4096, 4128          # 32 outputs of the wide layer ...
    rows, chunk = 32768, 4096    # ... x 32768 rows = 1.05e6 outputs
    layer = pkg.Layer.random(n_in, n_out, G, seed=55, out_range=(ob, oe))
    assert layer.plan(rows)["mode"] in ("staged", "fused")
    P = layer.read_table()
    worst, n = _scan(torch, pkg, ref, layer, P, n_in, rows, chunk, seed=9)
    # the same scan with one running sum (pair blocks off), for the record
    monkeypatch.setenv("LMKAN_B200_PAIR_BLOCK", "0")
    plain = pkg.Layer.random(n_in, n_out, G, seed=55, out_range=(ob, oe))
    worst_plain, _ = _scan(torch, pkg, ref, plain, P, n_in, rows // 4, chunk, seed=9)
    rec = {"outputs": n, "max_mixed_err": worst, "margin": TOL / worst,
           "max_mixed_err_single_sum_first_quarter": worst_plain, "oracle": "reference" if ref else "port"}
    print("cfg5 accumulation scan:", json.dumps(rec))
    out = os.environ.get("LMKAN_B200_ACCURACY_OUT")
    if out:
        with open(out, "w") as f:
            json.dump(rec, f, indent=1)
    assert n >= 1_000_000
    assert worst * 1.5 <= TOL, f"margin {TOL / worst:.2f}x < 1.5x (max mixed err {worst:.3e})"


def test_pair_block_edges_parity(torch, pkg, oracle, monkeypatch):
    """Pair blocks forced small on small layers (block boundaries inside and at
    the end of the pair range, ragged outputs, fp64 I/O, narrow layers): parity
    with the oracle and bitwise agreement across kernel modes."""
    rng = np.random.default_rng(4)
    for n_in, n_out, G, rows, blk in [(40, 24, 8, 3000, "4"), (64, 64, 12, 777, "32"), (46, 3, 8, 500, "4"),
                                      (30, 17, 6, 2049, "8")]:
        monkeypatch.setenv("LMKAN_B200_PAIR_BLOCK", blk)
        P = (rng.standard_normal((G + 1, G + 1, n_in // 2, n_out)) / np.sqrt(n_in // 2)).astype(np.float32)
        X = rng.standard_normal((rows, n_in)).astype(np.float32)
        outs = []
        for mode in ("staged", "fused"):
            monkeypatch.setenv("LMKAN_B200_MODE", mode)
            layer = pkg.Layer.from_host(n_in, n_out, G, P.astype(np.float64), 0.7)
            Y = layer.forward(torch.from_numpy(X).cuda()).cpu().numpy()
            outs.append(Y)
            Y64 = layer.forward(torch.from_numpy(X).double().cuda()).cpu().numpy()
            assert np.array_equal(Y64, Y.astype(np.float64))  # fp64 I/O == fp32 I/O bitwise
        monkeypatch.delenv("LMKAN_B200_MODE")
        monkeypatch.setenv("LMKAN_B200_NARROW", "0")  # narrow layers: the general kernel agrees bitwise
        wide = pkg.Layer.from_host(n_in, n_out, G, P.astype(np.float64), 0.7)
        outs.append(wide.forward(torch.from_numpy(X).cuda()).cpu().numpy())
        monkeypatch.delenv("LMKAN_B200_NARROW")
        assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
        ref = oracle.forward(G, P.astype(np.float64), X.astype(np.float64), 0.7)
        import pyoracle
        assert pyoracle.mixed_err(outs[0], ref).max() <= TOL
