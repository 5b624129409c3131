"""Generate tests/golden/golden.npz from the REFERENCE ITSELF.

Runs the unmodified reference headers (/root/reference/proj/include, compiled
into oracle/_ref/liblmkan_ref.so by oracle/Makefile via oracle/ref_shim.cpp).
Run in the build container (the GPU box has no /root/reference):

    make -C oracle && python tests/golden/make_golden.py

Contents (all produced by reference code paths):
  grid_G{G}_points / _inv         build_grid (grid.hpp:44-68)
  thr_G{G}_f32 / _f64             min{x : interval_index(x) >= k}, each threshold
                                  checked against the reference interval_index
                                  at t and at the next-lower value (grid.hpp:72-75)
  loc_G{G}_X / _i1 / _i2 / _w     row_preambles (layer.hpp:96-101) on normal,
                                  Cauchy and edge-case inputs
  fwd_{k}_*                       lmkan_forward (layer.hpp:108-134) cases
  init_{k}_P                      init_layer tables (layer.hpp:69-86)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pyoracle  # noqa: E402

GS = [3, 4, 5, 8, 12, 13, 16, 20, 28, 32, 40]
FWD_CASES = [  # (n_in, n_out, G, rows, gamma, xscale) — shapes from test_layer.cpp plus config shapes
    (2, 1, 5, 64, 1.0, 1.0), (6, 5, 3, 64, 0.8, 1.5), (6, 5, 12, 64, 0.8, 1.5), (8, 3, 4, 32, 0.6, 2.0),
    (8, 6, 12, 33, 0.9, 1.0), (64, 64, 8, 64, 1.0, 1.0), (12, 16, 28, 32, 1.0, 1.0), (36, 16, 16, 32, 1.0, 1.0),
]
INIT_CASES = [(4, 3, 4, 123, -1.0), (4, 3, 4, 124, -1.0), (6, 5, 3, 80, -1.0), (64, 8, 8, 7, 0.25)]


def main():
    ref = pyoracle.Ref()
    port = pyoracle.Port()
    out = {}
    rng = np.random.default_rng(20250907)
    for G in GS:
        pts, inv = ref.build_grid(G)
        out[f"grid_G{G}_points"], out[f"grid_G{G}_inv"] = pts, inv
        t32 = port.thresholds_f32(G)
        t64 = port.thresholds_f64(G)
        for k in range(1, G):  # pin each threshold on the reference function itself
            lo32 = np.nextafter(t32[k - 1], np.float32(-np.inf), dtype=np.float32)
            assert ref.interval_index(G, float(t32[k - 1]))[0] >= k > ref.interval_index(G, float(lo32))[0]
            assert ref.interval_index(G, t64[k - 1])[0] >= k > ref.interval_index(G, np.nextafter(t64[k - 1], -np.inf))[0]
        out[f"thr_G{G}_f32"], out[f"thr_G{G}_f64"] = t32, t64
        edge = np.array([0.0, -0.0, 1e-300, -1e-300, -2.0 ** -54, -2.0 ** -53, 2.0 ** -54, np.inf, -np.inf, np.nan,
                         1e308, -1e308, 100.0, -100.0, 0.1, -np.log(2.0)] + list(pts) + list(t64))
        X = np.concatenate([rng.standard_normal(256), np.tan(np.pi * (rng.random(256) - 0.5)), edge])
        if X.size % 2:
            X = np.append(X, 0.5)
        X = X.reshape(-1, 2)
        i1, i2, w = ref.locate(G, X)
        out[f"loc_G{G}_X"], out[f"loc_G{G}_i1"], out[f"loc_G{G}_i2"], out[f"loc_G{G}_w"] = X, i1, i2, w
    for k, (n_in, n_out, G, rows, gamma, xs) in enumerate(FWD_CASES):
        P = (rng.standard_normal((G + 1, G + 1, n_in // 2, n_out)) / np.sqrt(n_in // 2)).astype(np.float32)
        X = (rng.standard_normal((rows, n_in)) * xs).astype(np.float32)
        Y = ref.forward(G, P.astype(np.float64), X.astype(np.float64), gamma, workers=3)
        out[f"fwd_{k}_shape"] = np.array([n_in, n_out, G, rows])
        out[f"fwd_{k}_gamma"] = np.array(gamma)
        out[f"fwd_{k}_P"], out[f"fwd_{k}_X"], out[f"fwd_{k}_Y"] = P, X, Y
    for k, (n_in, n_out, G, seed, sc) in enumerate(INIT_CASES):
        out[f"init_{k}_args"] = np.array([n_in, n_out, G, seed, sc])
        out[f"init_{k}_P"] = ref.init_table(n_in, n_out, G, seed, sc)
    path = os.path.join(HERE, "golden.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes,", len(out), "arrays")


if __name__ == "__main__":
    main()
