"""Training-path timing: lmkan_backward (layer.hpp:141-202) on the B200 vs the
reference's own CPU lmkan_backward (oracle/_ref, LMKAN_THREADS = nproc) on a
bounded row sample. Usage: python tools/bench_backward.py
Prints one JSON line per shape (rows/s; the GPU result is bit-identical to the
reference at workers = 1, the CPU baseline uses all host threads)."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_2509_07103_b200 as pkg  # noqa: E402
import pyoracle  # noqa: E402

SHAPES = [  # (name, n_in, n_out, G, rows)
    ("student hidden layer 32->32, G=12", 32, 32, 12, 65536),
    ("methane hidden layer 128->128, G=28", 128, 128, 28, 65536),
    ("cfg1 layer 64->64, G=8", 64, 64, 8, 1024),
    ("cfg2 layer 1024->1024, G=16", 1024, 1024, 16, 4096),
]


def main():
    cores = os.cpu_count() or 1
    os.environ["LMKAN_THREADS"] = str(cores)
    ref = pyoracle.Ref()
    for name, n_in, n_out, G, rows in SHAPES:
        rng = np.random.default_rng(0)
        P = rng.standard_normal((G + 1, G + 1, n_in // 2, n_out)) / np.sqrt(n_in // 2)
        X = rng.standard_normal((rows, n_in))
        dY = rng.standard_normal((rows, n_out))
        layer = pkg.Layer.from_host(n_in, n_out, G, P, 1.0)
        Pd, Xd, dYd = (torch.from_numpy(a).cuda() for a in (P, X, dY))
        dP = torch.zeros_like(Pd)
        dX = torch.empty_like(Xd)
        s = torch.cuda.current_stream()
        for _ in range(2):
            layer.backward(Pd, Xd, dYd, dP=dP)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        K = 5 if rows * n_in * n_out < 1e10 else 2
        torch.cuda.synchronize()
        a.record(s)
        for _ in range(K):
            layer.backward(Pd, Xd, dYd, dP=dP)
        b.record(s)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / K
        # reference CPU on a bounded sample
        sub = min(rows, 4096)
        t0 = time.perf_counter()
        reps = 0
        while True:
            ref.backward(G, P, X[:sub], dY[:sub], 1.0, workers=cores)
            reps += 1
            if time.perf_counter() - t0 > 3.0:
                break
        cpu = sub * reps / (time.perf_counter() - t0)
        del dX
        print(json.dumps({"workload": f"lmkan_backward {name}, batch {rows}", "gpu_rows_per_s": rows / (ms / 1e3),
                          "gpu_ms": ms, "cpu_rows_per_s": cpu, "cpu_threads": cores,
                          "cpu_sample": f"{sub} rows x {reps} runs (reference lmkan_backward, workers=nproc)",
                          "speedup": rows / (ms / 1e3) / cpu}), flush=True)


if __name__ == "__main__":
    main()
