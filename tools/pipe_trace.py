"""Timeline of the host pipeline (LMKAN_B200_PIPE_TRACE) for the cfg4 conv and
the cfg2 layer host entries: H2D / kernels / D2H per chunk of the last call.

python tools/pipe_trace.py [cfg4|cfg2]   (the trace goes to stderr)
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2509_07103_b200 as pkg  # noqa: E402


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
    if which == "cfg4":
        layer = pkg.Layer.random(144, 16, 16, seed=1)
        X = torch.randn((256, 34, 34, 16)).pin_memory()
        Y = torch.empty((256 * 32 * 32, 16)).pin_memory()
        call = lambda: layer.conv_forward_host_ptr(X.data_ptr(), 256, 34, 34, 16, 3, 1, Y.data_ptr())  # noqa: E731
    else:
        layer = pkg.Layer.random(1024, 1024, 16, seed=1)
        X = torch.randn((65536, 1024)).pin_memory()
        Y = torch.empty((65536, 1024)).pin_memory()
        call = lambda: layer.forward_host_ptr(X.data_ptr(), Y.data_ptr(), 65536)  # noqa: E731
    for _ in range(5):
        call()
    t = time.perf_counter()
    for _ in range(20):
        call()
    print(f"{which}: {(time.perf_counter() - t) / 20 * 1e3:.4f} ms per call (untraced)", flush=True)
    os.environ["LMKAN_B200_PIPE_TRACE"] = "1"
    for _ in range(3):
        call()
        print("---", file=sys.stderr, flush=True)


if __name__ == "__main__":
    main()
