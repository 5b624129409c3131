"""Forward time of one layer shape under the current environment (planner
knobs such as LMKAN_B200_OT take effect at layer creation).

python tools/ubench_shape.py n_in n_out G rows [reps]  -> one JSON line
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2509_07103_b200 as pkg  # noqa: E402


def main():
    n_in, n_out, G, rows = (int(a) for a in sys.argv[1:5])
    reps = int(sys.argv[5]) if len(sys.argv) > 5 else 20
    layer = pkg.Layer.random(n_in, n_out, G, seed=1)
    X = torch.randn((rows, n_in), device="cuda")
    Y = torch.empty((rows, n_out), device="cuda")
    flush = torch.empty(64 << 20, device="cuda")
    s = torch.cuda.current_stream()
    for _ in range(3):
        layer.forward_into(X, Y, s)
    ms = []
    for i in range(reps):
        flush.fill_(float(i))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        layer.forward_into(X, Y, s)
        b.record(s)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    ms.sort()
    print(json.dumps({"shape": [n_in, n_out, G, rows], "ms_median": ms[len(ms) // 2], "plan": layer.plan(rows),
                      "env_ot": os.environ.get("LMKAN_B200_OT")}))


if __name__ == "__main__":
    main()
