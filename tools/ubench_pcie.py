"""PCIe copy rates on the box: pinned H2D alone, D2H alone, and both at once
on separate streams (is the link full duplex for the host pipeline?), at the
cfg4 e2e sizes (18.9 MB images in, 16.8 MB outputs back) and in chunks.

python tools/ubench_pcie.py  -> one JSON line per case
"""
import json
import time

import torch


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


def main():
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    n_in, n_out = 18939904, 16777216
    h_in = torch.empty(n_in, dtype=torch.uint8, pin_memory=True)
    h_out = torch.empty(n_out, dtype=torch.uint8, pin_memory=True)
    d_in = torch.empty(n_in, dtype=torch.uint8, device="cuda")
    d_out = torch.empty(n_out, dtype=torch.uint8, device="cuda")

    def h2d():
        with torch.cuda.stream(s_in):
            d_in.copy_(h_in, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s_out):
            h_out.copy_(d_out, non_blocking=True)

    def both():
        h2d()
        d2h()

    t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
    print(json.dumps({"case": "whole", "h2d_ms": t1 * 1e3, "h2d_gbs": n_in / t1 / 1e9, "d2h_ms": t2 * 1e3,
                      "d2h_gbs": n_out / t2 / 1e9, "both_ms": t3 * 1e3, "sum_ms": (t1 + t2) * 1e3}))
    for chunks in (2, 4, 8, 16):
        ci, co = n_in // chunks, n_out // chunks

        def h2d_c():
            with torch.cuda.stream(s_in):
                for c in range(chunks):
                    d_in[c * ci:(c + 1) * ci].copy_(h_in[c * ci:(c + 1) * ci], non_blocking=True)

        def d2h_c():
            with torch.cuda.stream(s_out):
                for c in range(chunks):
                    h_out[c * co:(c + 1) * co].copy_(d_out[c * co:(c + 1) * co], non_blocking=True)

        def both_c():
            h2d_c()
            d2h_c()

        t1, t2, t3 = timed(h2d_c), timed(d2h_c), timed(both_c)
        print(json.dumps({"case": f"{chunks} chunks", "h2d_ms": t1 * 1e3, "d2h_ms": t2 * 1e3, "both_ms": t3 * 1e3}))


if __name__ == "__main__":
    main()
