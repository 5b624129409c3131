"""LMK1 model container (serialize.hpp:185-301) and the fused-model chain
(model_infer, model.hpp:268-315) on the B200 path.

Fixtures under tests/golden/lmk1/ were written BY THE REFERENCE
(tests/golden/make_lmk1.py: build_student -> fuse_model -> save_model), and
golden.json holds the reference's own model_infer outputs and its load_model
verdict (exception type + message) on every corruption in lmk1_variants.py.
"""
import json
import os

import numpy as np
import pytest

import lmk1_variants

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden", "lmk1")
TOL = 1e-5


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(GOLD, "golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def pkg():
    import paper_2509_07103_b200 as p
    return p


# ------------------------------------------------------------------ host only
def test_reference_files_validate(pkg, golden):
    for name, verdict in golden["files"].items():
        info = pkg.lmk1_inspect(os.path.join(GOLD, name))
        assert info["blocks"] == verdict["ok"], name
        assert info["pure_lookup"] == name.startswith("pure"), name
        assert info["dtype"] == ("f32" if "f32" in name else "f64")


# Messages that embed nlohmann's own exception text: compare up to the prefix.
_NLOHMANN_PREFIX = ("load_model: header is not valid JSON:", "load_model: malformed block metadata:")


@pytest.mark.parametrize("case", [
    "empty", "bad_magic", "trunc_len", "trunc_header", "bad_json", "bad_format", "bad_version", "bad_dtype",
    "unknown_block", "bad_mode", "bad_G", "missing_key", "manifest_order", "manifest_short", "bytes_mismatch",
    "trunc_payload", "trailing"])
def test_corruption_verdicts_match_reference(pkg, golden, tmp_path, case):
    """Same exception class (FormatError / invalid_argument) and message as the
    reference's load_model on the same corrupted bytes."""
    base = open(os.path.join(GOLD, "pure_f64.lmk1"), "rb").read()
    blob = lmk1_variants.variants(base)[case]
    p = tmp_path / f"{case}.lmk1"
    p.write_bytes(blob)
    ref = golden["cases"][case]
    expect = {"FormatError": pkg.FormatError, "invalid_argument": ValueError}[ref["error"]]
    with pytest.raises(expect) as ei:
        pkg.lmk1_inspect(str(p))
    msg = ei.value.msg if isinstance(ei.value, pkg.LmkanError) else str(ei.value)
    pre = next((x for x in _NLOHMANN_PREFIX if ref["message"].startswith(x)), None)
    if pre:
        assert msg.startswith(pre), (msg, ref["message"])
    else:
        assert msg == ref["message"]


def test_missing_file(pkg, tmp_path):
    with pytest.raises(pkg.FormatError, match="load_model: cannot open"):
        pkg.lmk1_inspect(str(tmp_path / "nope.lmk1"))


def test_block_metadata_matches_header(pkg):
    # relu_first student (train.hpp:106-140): first layer 'linear', then
    # 'relu_first'; batch norms after every layer but the last
    path = os.path.join(GOLD, "student.lmk1")
    blocks = [pkg.lmk1_block(path, i) for i in range(3)]
    assert [b["mode"] for b in blocks] == ["linear", "relu_first", "relu_first"]
    assert [b["bn"] for b in blocks] == [True, True, False]
    assert [(b["n_in"], b["n_out"], b["G"]) for b in blocks] == [(6, 8, 8), (8, 8, 8), (8, 3, 8)]
    assert all(abs(b["gamma"] - 0.7) < 1e-15 for b in blocks)
    pure = [pkg.lmk1_block(os.path.join(GOLD, "pure_f64.lmk1"), i) for i in range(3)]
    assert all(b["mode"] == "none" and not b["bn"] and b["gamma"] == 1.0 for b in pure)
    with pytest.raises(ValueError):
        pkg.lmk1_block(path, 3)


def test_p_offsets_locate_the_payload(pkg):
    """p_offset points at the block's P tensor; reading it with numpy gives the
    table the reference saved (used by the GPU tests as the expected table)."""
    path = os.path.join(GOLD, "pure_f64.lmk1")
    raw = open(path, "rb").read()
    b0 = pkg.lmk1_block(path, 0)
    n = (b0["G"] + 1) ** 2 * (b0["n_in"] // 2) * b0["n_out"]
    P = np.frombuffer(raw, "<f8", count=n, offset=b0["p_offset"])
    assert np.isfinite(P).all() and np.abs(P).max() > 0


@pytest.mark.parametrize("name,what", [("student.lmk1", "preconditioned"), ("mlp.lmk1", "batch-norm")])
def test_non_fused_models_rejected(pkg, name, what):
    """The B200 path serves fused pure-lookup models; others are refused before
    any device work (also without a GPU)."""
    with pytest.raises(pkg.UnsupportedModelError, match=what):
        pkg.load_model(os.path.join(GOLD, name))


# ------------------------------------------------------------------ GPU
def _payload_table(path, pkg, block):
    b = pkg.lmk1_block(path, block)
    n = (b["G"] + 1) ** 2 * (b["n_in"] // 2) * b["n_out"]
    dt = "<f4" if pkg.lmk1_inspect(path)["dtype"] == "f32" else "<f8"
    P = np.frombuffer(open(path, "rb").read(), dt, count=n, offset=b["p_offset"]).astype(np.float64)
    return b, P.reshape(b["G"] + 1, b["G"] + 1, b["n_in"] // 2, b["n_out"])


@pytest.mark.gpu
@pytest.mark.parametrize("name,key", [("pure_f64.lmk1", "Y_f64"), ("pure_f32.lmk1", "Y_f32")])
def test_load_model_infer_matches_reference(pkg, golden, name, key):
    """load_model + model_infer on the device vs the reference's own
    model_infer(load_model(file)) outputs; tables equal the payload rounded to fp32."""
    path = os.path.join(GOLD, name)
    model = pkg.load_model(path)
    assert (model.n_blocks, model.in_dim, model.out_dim) == (3, 6, 3)
    for i in range(3):
        b, P = _payload_table(path, pkg, i)
        got = model.layer(i).read_table()
        assert np.array_equal(got, P.astype(np.float32).astype(np.float64)), i
    X = np.array(golden["io"]["X"]).reshape(16, 6)
    ref = np.array(golden["io"][key]).reshape(16, 3)
    for Y in (pkg.model_infer(model, X), model.infer_host(X.astype(np.float32)).astype(np.float64)):
        err = np.abs(Y - ref) / np.maximum(1.0, np.abs(ref))
        assert err.max() <= TOL, err.max()


@pytest.mark.gpu
def test_model_chain_graph_replay_bitwise(pkg):
    """Model.infer (device, side stream) = the layers run one by one, bitwise,
    on the eager first call and on CUDA-graph replays; new shapes re-capture."""
    import torch
    layers = [pkg.Layer.random(12, 128, 28, seed=1), pkg.Layer.random(128, 128, 28, seed=2),
              pkg.Layer.random(128, 1, 28, seed=3)]
    model = pkg.Model.from_layers(layers)
    st = torch.cuda.Stream()
    for rows in (3000, 70000, 3000):
        X = torch.randn((rows, 12), device="cuda")
        ref = X
        for lay in layers:
            ref = lay.forward(ref)
        Y = torch.empty((rows, 1), device="cuda")
        for _ in range(3):
            Y.fill_(float("nan"))
            with torch.cuda.stream(st):
                model.infer_into(X, Y, st)
            st.synchronize()
            assert torch.equal(Y, ref), rows


@pytest.mark.gpu
def test_layer_load_lmk1_output_slices(pkg):
    """Sharded load: output slices of one block straight from the file equal the
    corresponding columns of the full layer, bitwise."""
    import torch
    path = os.path.join(GOLD, "pure_f64.lmk1")
    full = pkg.Layer.load_lmk1(path, 1)
    X = torch.randn((500, 8), device="cuda")
    Y = full.forward(X)
    for ob, oe in [(0, 3), (3, 8), (5, 6)]:
        sl = pkg.Layer.load_lmk1(path, 1, out_range=(ob, oe))
        assert torch.equal(sl.forward(X), Y[:, ob:oe])
    with pytest.raises(ValueError):
        pkg.Layer.load_lmk1(path, 1, out_range=(4, 9))


@pytest.mark.gpu
def test_model_width_mismatch(pkg):
    import torch
    a, b = pkg.Layer.random(6, 8, 8, seed=1), pkg.Layer.random(10, 3, 8, seed=2)
    model = pkg.Model.from_layers([a, b])
    with pytest.raises(ValueError, match="precond_forward: expected width 10, got 8"):
        model.infer(torch.randn((4, 6), device="cuda"))


@pytest.mark.gpu
@pytest.mark.parametrize("rows", [777, 5000, 66000])
def test_fused_chain_records_bitwise(pkg, monkeypatch, rows):
    """Fused chain (each layer's epilogue writes the next layer's cell records,
    skipping that layer's K1 and its activation round trip): bitwise equal to
    the unfused chain and to the layers run one by one, for consecutive fusions
    and ragged row counts."""
    import torch
    dims = [(16, 64, 8), (64, 96, 12), (96, 64, 8), (64, 2, 8)]
    layers = [pkg.Layer.random(a, b, G, seed=20 + i) for i, (a, b, G) in enumerate(dims)]
    X = torch.randn((rows, 16), device="cuda")
    ref = X
    for lay in layers:
        ref = lay.forward(ref)
    st = torch.cuda.Stream()
    outs = []
    for fuse in ("1", "0"):
        monkeypatch.setenv("LMKAN_B200_CHAIN_FUSE", fuse)
        monkeypatch.setenv("LMKAN_B200_GRAPH", "0")
        model = pkg.Model.from_layers(layers)
        Y = torch.full((rows, 2), float("nan"), device="cuda")
        with torch.cuda.stream(st):
            model.infer_into(X, Y, st)
        st.synchronize()
        outs.append(Y)
    assert torch.equal(outs[0], ref) and torch.equal(outs[1], ref)


def _write_lmk1(path, blocks, dtype="f32"):
    """Minimal LMK1 writer for pure-lookup models (serialize.hpp:109-183 format:
    magic, u32 LE header length, JSON header, LE payload P[i1][i2][pair][out])."""
    elem = 4 if dtype == "f32" else 8
    hb = {"blocks": [], "dtype": dtype, "format": "LMK1", "tensors": [], "version": 1}
    payload = []
    for i, (n_in, n_out, G, P) in enumerate(blocks):
        hb["blocks"].append({"G": G, "gamma": 1.0, "mode": "none", "n_in": n_in, "n_out": n_out, "type": "lmkan"})
        hb["tensors"].append({"bytes": P.size * elem, "name": f"block{i}.P", "shape": list(P.shape)})
        payload.append(np.ascontiguousarray(P, "<f4" if elem == 4 else "<f8").tobytes())
    h = json.dumps(hb, separators=(",", ":")).encode()
    with open(path, "wb") as f:
        f.write(b"LMK1" + len(h).to_bytes(4, "little") + h + b"".join(payload))


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_lmk1_multichunk_stream(pkg, tmp_path, dtype):
    """A block larger than the 64 MB staging chunk (several double-buffered
    chunks, chunk boundaries inside a node): the device table equals the
    payload rounded to fp32, for the whole layer and for an output slice."""
    rng = np.random.default_rng(3)
    n_in, n_out, G = 512, 520, 16  # 289 * 256 * 520 values: 154 MB f32, 308 MB f64
    P = rng.standard_normal((G + 1, G + 1, n_in // 2, n_out)).astype(np.float32).astype(np.float64)
    path = str(tmp_path / "big.lmk1")
    _write_lmk1(path, [(n_in, n_out, G, P), (n_out, 4, 8, rng.standard_normal((9, 9, n_out // 2, 4)))], dtype)
    assert pkg.lmk1_inspect(path)["blocks"] == 2
    lay = pkg.Layer.load_lmk1(path, 0)
    want = P.astype(np.float32).astype(np.float64)
    for pb, pe in [(0, 40), (200, 256)]:
        assert np.array_equal(lay.read_table(pb, pe), want[:, :, pb:pe, :])
    sl = pkg.Layer.load_lmk1(path, 0, out_range=(100, 333))
    assert np.array_equal(sl.read_table(10, 30), want[:, :, 10:30, 100:333])


@pytest.mark.gpu
def test_model_graph_recaptures_after_gamma_change(pkg):
    """A captured chain bakes gamma into its kernel parameters: changing a
    layer's gamma must not replay the stale graph."""
    import torch
    layers = [pkg.Layer.random(16, 32, 8, seed=1), pkg.Layer.random(32, 8, 8, seed=2)]
    model = pkg.Model.from_layers(layers)
    st = torch.cuda.Stream()
    X = torch.randn((1000, 16), device="cuda")
    Y = torch.empty((1000, 8), device="cuda")
    for _ in range(2):
        with torch.cuda.stream(st):
            model.infer_into(X, Y, st)
    st.synchronize()
    base = Y.clone()
    layers[1].set_gamma(0.5)
    with torch.cuda.stream(st):
        model.infer_into(X, Y, st)
    st.synchronize()
    assert torch.allclose(Y, 0.5 * base, rtol=1e-6, atol=1e-7)
