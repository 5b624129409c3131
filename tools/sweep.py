"""Kernel-variant sweep on one GPU (in-process; LMKAN_B200_* env vars are read
per call). Usage: python tools/sweep.py [config] — prints one line per variant."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2509_07103_b200 as pkg  # noqa: E402


def time_layer(layers, X, acts, iters=10):
    """Device time per step; with SWEEP_GRAPH=1 the steps are captured in one
    CUDA graph (no host launch gaps: the kernels' own time for tiny batches)."""
    graph = os.environ.get("SWEEP_GRAPH") == "1"
    s = torch.cuda.current_stream()

    def step():
        st = torch.cuda.current_stream()
        cur = X
        for lay, out in zip(layers, acts):
            lay.forward_into(cur, out, st)
            cur = out
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    if graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(iters):
                step()
        g.replay()
        torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(s)
    if graph:
        g.replay()
    else:
        for _ in range(iters):
            step()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def main():
    cfgn = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    cfg = bench.CONFIGS[cfgn]
    sw = os.environ.get("SWEEP", "[]")
    if sw.endswith(".json"):
        sw = open(sw).read()
    variants = json.loads(sw) or [
        {"LMKAN_B200_MODE": m, "LMKAN_B200_RT": rt, "LMKAN_B200_NBUF": nb}
        for m in ("staged", "fused") for rt in ("16", "8") for nb in ("2", "1", "3")]
    G, B = cfg["G"], cfg["batch"]
    X = torch.randn((B, cfg["layers"][0][0]), device="cuda")
    shard = int(os.environ.get("SWEEP_SHARD", "0"))
    acts = [torch.empty((B, o // shard if shard else o), device="cuda") for _, o in cfg["layers"]]
    ot_cache = {}
    for v in variants:
        for k in [k for k in os.environ if k.startswith("LMKAN_B200_")]:
            os.environ.pop(k, None)
        os.environ.update(v)
        key = v.get("LMKAN_B200_OT", "")
        if key not in ot_cache:
            shard = int(os.environ.get("SWEEP_SHARD", "0"))  # output-sharded layer: shard 0 of SWEEP_SHARD
            ot_cache.clear()
            ot_cache[key] = [pkg.Layer.random(a, b, G, seed=1000 + i,
                                              out_range=(0, b // shard) if shard else None)
                             for i, (a, b) in enumerate(cfg["layers"])]
        layers = ot_cache[key]
        try:
            ms = time_layer(layers, X, acts)
            plan = layers[0].plan(B)
            print(json.dumps({"variant": v, "ms": round(ms, 4), "samples_per_s": B / ms * 1e3, "plan": plan}),
                  flush=True)
        except Exception as e:  # noqa: BLE001
            print(json.dumps({"variant": v, "error": str(e)}), flush=True)


if __name__ == "__main__":
    main()
