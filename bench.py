#!/usr/bin/env python3
"""lmKAN layer forward throughput on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config 1..7]  (5: output-sharded wide layer, 6 / 7: conv stages 2 / 3)

One step = one lmkan forward over one batch of the workload. Default workload
(N=1) is BASELINE.json configs[1] ("cfg2"): a single layer 1024 -> 1024, G=16,
batch 65536, fp32, synthetic N(0,1) inputs and an N(0, 1/512) table generated on
the device. Batch rows are independent (layer.hpp:116-133), so under torchrun
every rank runs its own 65536-row batch against a replica of the table (weak
scaling, no collective); timing is the max over ranks of CUDA-event time.

Printed JSON line (rank 0): value = samples/s of the whole job (device-resident
inputs), e2e = the same through the public host entry point
(lmkan_b200_forward_host_f32: pinned host X in, host Y out, copies pipelined
with the kernel), roofline = the fused kernel's algorithmic bytes per launch /
its event-timed duration vs the measured HBM copy peak, cpu_baseline = the
reference's own lmkan_forward (oracle/_ref, compiled from /root/reference) on
this host's cores over a bounded row sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    1: dict(name="cfg1: lmKAN layer 64->64, G=8, batch 1024", layers=[(64, 64)], G=8, batch=1024, small=True),
    2: dict(name="cfg2: lmKAN layer 1024->1024, G=16, batch 65536", layers=[(1024, 1024)], G=16, batch=65536),
    3: dict(name="cfg3: methane pure-lookup chain 12->128->128->1, G=28, batch 1048576",
            layers=[(12, 128), (128, 128), (128, 1)], G=28, batch=1 << 20),
    4: dict(name="cfg4: lmKAN 3x3 conv (implicit im2col), 144->16, G=16, 256 images 32x32x16 (zero-padded 34x34)",
            layers=[(144, 16)], G=16, batch=262144, conv=dict(N=256, H=34, W=34, C=16, k=3, s=1)),
}
# config 4's later ResNet stages, reported beside it
CONFIGS[6] = dict(name="cfg4 stage 2: lmKAN 3x3 conv (implicit im2col), 288->32, G=16, 256 images 16x16x32 (zero-padded 18x18)",
                  layers=[(288, 32)], G=16, batch=65536, conv=dict(N=256, H=18, W=18, C=32, k=3, s=1))
CONFIGS[7] = dict(name="cfg4 stage 3: lmKAN 3x3 conv (implicit im2col), 576->64, G=16, 256 images 8x8x64 (zero-padded 10x10)",
                  layers=[(576, 64)], G=16, batch=16384, conv=dict(N=256, H=10, W=10, C=64, k=3, s=1))
CONFIGS[5] = dict(name="cfg5: wide lmKAN layer 8192->8192, G=32, batch 262144, output-sharded",
                  layers=[(8192, 8192)], G=32, batch=262144, out_sharded=True)
L2_BYTES = 126 << 20
METRIC = "lmKAN layer fwd samples/s at 1/2/4/8 B200; achieved GB/s vs HBM roofline"


def b_alg(n_in: int, n_out: int) -> int:
    """Algorithmic bytes per sample per layer: 4 fp32 table
    coefficients per 2D function + the X row + the Y row."""
    return 8 * n_in * n_out + 4 * (n_in + n_out)


def fma_per_row(n_in: int, n_out: int) -> int:
    return 2 * n_in * n_out  # costs.hpp:14-23


def smem_ceiling(fma_per_row: float, sm_mhz, kernel_ms: float, rows: int) -> dict:
    """Gather ceiling: 148 SMs x 32 FMA/clk (128 B/clk of shared-memory reads
    at 4 B per coefficient) at the measured SM clock, in rows/s, and the
    kernel's fraction of it."""
    mhz = float(sm_mhz or 1965.0)
    fma_s = 148 * 32 * mhz * 1e6
    ceil_rows = fma_s / fma_per_row
    achieved = rows / (kernel_ms / 1e3)
    return {"fma_per_s": fma_s, "rows_per_s": ceil_rows, "achieved_rows_per_s": achieved,
            "frac": achieved / ceil_rows, "sm_mhz": mhz}


def roofline_levels(achieved_gbs: float, fma_per_s: float, hbm_gbs: float, sm_mhz) -> dict:
    """B_alg-based GB/s against HBM (MEASURED_PEAKS.json), L2 (tools/ubench_l2.cu,
    profiles/r1_ubench_l2.json), the shared-memory port (148 x 128 B/clk) and
    FMA/s against the FP32 pipe (148 x 128 FMA/clk), at the measured SM clock."""
    mhz = float(sm_mhz or 1965.0)
    l2 = None
    try:
        with open(os.path.join(ROOT, "profiles", "r1_ubench_l2.json")) as f:
            l2 = float(json.load(f)["l2_read_gbs"])
    except Exception:
        pass
    smem = 148 * 128 * mhz * 1e6 / 1e9
    fp32 = 148 * 128 * mhz * 1e6
    out = {"hbm": {"peak_gbs": hbm_gbs, "frac": achieved_gbs / hbm_gbs},
           "smem": {"peak_gbs": smem, "frac": achieved_gbs / smem},
           "fp32_fma": {"peak_fma_per_s": fp32, "frac": fma_per_s / fp32}}
    if l2:
        out["l2"] = {"peak_gbs": l2, "frac": achieved_gbs / l2, "source": "profiles/r1_ubench_l2.json"}
    return out


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def load_traffic(cfg: int):
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(f"cfg{cfg}", {}).get("dram_bytes_per_launch")
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.samples = []
        self.window = None
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(gpu), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()
        t0 = time.time()
        while not self.samples and time.time() - t0 < 5:
            time.sleep(0.02)

    def _read(self):
        for line in self.p.stdout:
            self.samples.append((time.time(), [x.strip() for x in line.split(",")]))

    def begin(self):
        self.window = [time.time(), None]

    def end(self):
        time.sleep(0.12)
        self.window[1] = time.time()

    def summary(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        t0, t1 = self.window
        win = [s for t, s in self.samples if t0 <= t <= t1] or [s for t, s in self.samples if t >= t0][:3]
        if not win:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(s[1]) for s in win if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in win if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for s in win for n, v in zip(names, s[4:8]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(win)}


def config_dict(cfg: dict, ws: int, rank: int, shards: int, gather: str) -> dict:
    """The workload description, identical in both arms (b200 and reference)."""
    B = cfg["batch"]
    out_sharded = bool(cfg.get("out_sharded"))
    if out_sharded:
        par = (f"output-sharded over {shards} (this run: {ws} process(es); shard {rank % shards}"
               + ((", all-gather of Y columns fused into the epilogue (NVLink peer stores)" if gather == "fused"
                   else ", NCCL all-gather of Y columns") if ws > 1 else
                  ", no all-gather: single-rank shard measurement") + ")")
    else:
        par = f"dp{ws} (batch rows, no collective)"
    return {"workload": cfg["name"], "layers": cfg["layers"], "G": cfg["G"], "batch_per_gpu": B,
            "global_batch": B if out_sharded else ws * B, "parallelism": par}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ------------------------------------------------------------------- CPU reference
def cpu_reference(cfg: dict, tables, step_s: float = 0.5, steps: int = 0, warmup: int = 0, budget_s: float = 12.0):
    """The reference's own lmkan_forward (oracle/_ref/liblmkan_ref.so compiled
    from /root/reference) on this host, all cores (LMKAN_THREADS = nproc).
    A CPU step = one pass of the layer chain over a bounded row sample of the
    workload, sized (by doubling from 64 rows) to take about step_s seconds.
    steps > 0: exactly `warmup` untimed + `steps` timed steps (the reference
    arm); else as many timed steps as fit budget_s (3..20, the cpu_baseline
    leg). Returns dict(rows, step_times, cores, kind)."""
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    cores = os.cpu_count() or 1
    os.environ["LMKAN_THREADS"] = str(cores)
    try:
        ref = pyoracle.Ref()
        kind = "reference"
    except (FileNotFoundError, OSError):
        ref = None
        kind = "port"
    G = cfg["G"]
    rng = np.random.default_rng(1234)
    layers = []
    for (n_in, n_out), P in zip(cfg["layers"], tables):
        if ref is not None:
            layers.append(pyoracle.RefLayer(ref, n_in, n_out, G, P, 1.0))
        else:
            layers.append((n_in, n_out, P))
    port = pyoracle.Port() if ref is None else None

    def run_chain(rows):
        """Seconds spent inside lmkan_forward for one pass of the layer chain
        (Matrix construction / readback outside the timed region, like
        calling lmkan_forward with a pre-allocated Y)."""
        X = rng.standard_normal((rows, cfg["layers"][0][0])).astype(np.float32).astype(np.float64)
        spent = 0.0
        cur = X
        for lay in layers:
            if ref is not None:
                xm, ym = lay.make_io(cur)
                t_a = time.perf_counter()
                lay.run(xm, ym, 0)
                spent += time.perf_counter() - t_a
                cur = lay.read(ym, rows)
                lay.free_io(xm, ym)
            else:
                n_in, n_out, P = lay
                t_a = time.perf_counter()
                cur = port.forward(G, P, cur, 1.0, threads=cores)
                spent += time.perf_counter() - t_a
        return spent

    rows = 64
    while True:  # calibrate the sample: double until a pass takes >= step_s / 2
        dt = run_chain(rows)
        if dt >= step_s / 2 or rows >= cfg["batch"]:
            break
        rows = min(cfg["batch"], rows * 2)
    if steps <= 0:
        steps = int(max(3, min(20, budget_s / max(dt, 1e-6))))
        warmup = 1 if dt > 1.0 else 2
    for _ in range(warmup):
        run_chain(rows)
    ts = [run_chain(rows) for _ in range(steps)]
    for lay in layers:
        if ref is not None:
            lay.close()
    return dict(rows=rows, step_times=ts, cores=cores, kind=kind, warmup=warmup)


def host_cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS))
    ap.add_argument("--precision", type=int, default=32, choices=[32, 64],
                    help="64: reference-precision layers (fp64 table and accumulation, bit-identical to the "
                         "reference forward; single dense layers only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--gather", default="fused", choices=["fused", "nccl"],
                    help="config 5 under torchrun: all-gather of the output columns fused into the gather "
                         "kernel's epilogue (NVLink peer stores + device barrier) or a separate NCCL all-gather")
    ap.add_argument("--shards", type=int, default=0,
                    help="config 5: number of output shards (default: world size); with one process, "
                         "measures shard 0 of K (what each of K GPUs computes) without the all-gather")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # self-launch: one process per GPU through torchrun on this node (the
        # driver may also launch bench.py under torchrun itself)
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        os.execvp(sys.executable, [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                                   f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
                                   "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]])
    ws, rank, local = dist_env()
    cfg = CONFIGS[args.config]

    if args.impl == "reference":
        if rank != 0:
            return
        reference_arm(args, cfg, ws)
        return

    import numpy as np
    import torch
    import paper_2509_07103_b200 as pkg

    # LMKAN_B200_BENCH_SHARE_GPU=1: a plumbing dry run of the multi-rank paths
    # on a box with fewer GPUs than ranks (ranks share devices, gloo instead of
    # NCCL, which refuses two ranks on one GPU); never a measurement
    share = os.environ.get("LMKAN_B200_BENCH_SHARE_GPU") == "1"
    if share:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    G = cfg["G"]
    B = cfg["batch"]
    out_sharded = bool(cfg.get("out_sharded"))
    peers = None
    Yfull = None
    shards = (args.shards or ws) if out_sharded else 1
    if out_sharded:
        from paper_2509_07103_b200 import sharding
        n_in0, n_out0 = cfg["layers"][0]
        ob, oe = sharding.shard_range(n_out0, rank % shards, shards, align=16)
        layers = [pkg.Layer.random(n_in0, n_out0, G, seed=1000, gamma=1.0, device=local, out_range=(ob, oe))]
        cfg = dict(cfg, layers=[(n_in0, oe - ob)])  # this rank's local layer
        Yfull = torch.empty((B, n_out0), device=f"cuda:{local}") if ws > 1 else None
        # all-gather of the column shards: fused into the gather kernel's
        # epilogue (NVLink stores into every rank's Y + device barrier), or NCCL
        peers = sharding.PeerGather(B, n_out0, local) if ws > 1 and args.gather == "fused" else None
    elif args.precision == 64:
        if len(cfg["layers"]) != 1 or cfg.get("conv"):
            raise SystemExit("--precision 64: single dense layer configs only (1, 2)")
        n_in, n_out = cfg["layers"][0]
        rng = np.random.default_rng(1000)
        P = rng.standard_normal((G + 1, G + 1, n_in // 2, n_out)) / np.sqrt(n_in // 2)
        layers = [pkg.Layer.from_host(n_in, n_out, G, P, 1.0, device=local, precision=64)]
        del P
    else:
        layers = [pkg.Layer.random(n_in, n_out, G, seed=1000 + i, gamma=1.0, device=local)
                  for i, (n_in, n_out) in enumerate(cfg["layers"])]
    gen = torch.Generator(device=f"cuda:{local}").manual_seed(1234 + rank)
    conv = cfg.get("conv")
    if conv:  # NHWC image batch; patch rows are formed on the fly (implicit im2col)
        X = torch.randn((conv["N"], conv["H"], conv["W"], conv["C"]), generator=gen, device=f"cuda:{local}",
                        dtype=torch.float32)
        X[:, 0] = 0
        X[:, -1] = 0
        X[:, :, 0] = 0
        X[:, :, -1] = 0  # zero padding ring of the 32x32 images
    else:
        X = torch.randn((B, cfg["layers"][0][0]), generator=gen, device=f"cuda:{local}", dtype=torch.float32)
    acts = [torch.empty((B, n_out), device=f"cuda:{local}", dtype=torch.float32) for _, n_out in cfg["layers"]]
    # Chains (and launch-bound tiny batches) run through the model API: one
    # device chain per step, replayed from a CUDA graph (needs a non-legacy
    # stream); single wide layers launch directly on the current stream.
    use_model = not conv and not out_sharded and args.precision == 32 and (len(layers) > 1 or bool(cfg.get("small")))
    model = pkg.Model.from_layers(layers) if use_model else None
    stream = torch.cuda.Stream() if use_model else torch.cuda.current_stream()
    K = args.steps
    # gather-kernel events per step and layer (the dominant kernel, timed alone
    # through lmkan_b200_forward_f32_timed); created by one record each
    gev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in layers]
           for _ in range(K)]
    for per in gev:
        for a, b in per:
            a.record(stream)
            b.record(stream)

    def step(i=None, src=None, eager=False):
        cur = X if src is None else src
        if model is not None and not eager:
            model.infer_into(cur, acts[-1], stream)
            return
        for li, (lay, out) in enumerate(zip(layers, acts)):
            if conv and li == 0:
                if i is not None:
                    gev[i][li][0].record(stream)
                lay.conv_forward(cur, conv["k"], conv["s"], Y=out.view(conv["N"], (conv["H"] - conv["k"]) // conv["s"] + 1,
                                                       (conv["W"] - conv["k"]) // conv["s"] + 1, -1),
                                 stream=stream)
                if i is not None:
                    gev[i][li][1].record(stream)
            elif peers is not None:  # fused: the epilogue writes every rank's full-width Y
                if i is not None:
                    gev[i][li][0].record(stream)
                peers.forward(lay, cur, ob, stream)
                if i is not None:
                    gev[i][li][1].record(stream)
            elif i is None:
                lay.forward_into(cur, out, stream)
            else:
                lay.forward_into_timed(cur, out, gev[i][li][0], gev[i][li][1], stream)
            cur = out
        if out_sharded and ws > 1 and peers is None:  # NCCL all-gather of the output-column shards
            sharding.gather_columns(acts[-1], n_out0, ws, rank, align=16, out=Yfull)

    # L2 policy: a step whose inputs, table and outputs fit the 126 MB L2 would
    # find them resident from the previous step, so such configs write a
    # 256 MB buffer between timed steps and time each step with its own events
    # (the flush outside them); larger working sets run back to back.
    work_bytes = X.numel() * 4 + sum(l.table_bytes for l in layers) + sum(a.numel() * 4 for a in acts)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=f"cuda:{local}") if work_bytes < L2_BYTES else None
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    sampler = ClockSampler(local) if rank == 0 else None
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)] if flush is not None else []
    if sampler:
        sampler.begin()
    start.record(stream)
    for i in range(K):
        if flush is not None:
            with torch.cuda.stream(stream):
                flush.fill_(float(i))
            sev[i][0].record(stream)
        step(None if model is not None else i)
        if flush is not None:
            sev[i][1].record(stream)
    stop.record(stream)
    torch.cuda.synchronize()
    if sampler:
        sampler.end()
    if peers is not None:
        peers.check()  # no rank timed out at the device barrier
    if model is not None:
        # graph replays carry no per-kernel events: time the gather kernels in
        # an eager pass of the same K steps right after the timed region
        for i in range(K):
            step(i, eager=True)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    elapsed_ms = start.elapsed_time(stop) if flush is None else sum(a.elapsed_time(b) for a, b in sev)
    gather_ms = [sum(a.elapsed_time(b) for a, b in per) for per in gev]
    t = torch.tensor([elapsed_ms], device=f"cuda:{local}")
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_ms = float(t.item())
    ms_per_step = elapsed_ms / K
    # batch-sharded configs: every rank runs its own B rows (weak scaling);
    # config 5: all ranks cooperate on the same B rows (strong scaling)
    value = (B if out_sharded else ws * B) / (ms_per_step / 1e3)
    kernel_ms = statistics.mean(gather_ms)  # gather kernel(s) of one step, event-timed on the launch stream
    launches_per_step = sum(l.plan(B)["launches"] for l in layers)

    # ---- e2e through the public API: pinned host input in, host result out.
    # Single dense layer: the synchronous host entry lmkan_b200_forward_host_f32;
    # chains / tiny batches: lmkan_b200_model_infer_host_f32; conv:
    # lmkan_b200_conv_forward_host_f32 (each pipelines H2D / kernels / D2H over
    # row or image chunks on two internal streams). Output-sharded: H2D, the
    # device step with its all-gather, D2H, then a host read of the result.
    e2e = None
    if not args.no_e2e:
        Xh = X.cpu().pin_memory()
        # the step's result: the full gathered Y when output-sharded over ranks
        Yres = (peers.Y if peers is not None else Yfull) if (out_sharded and ws > 1) else acts[-1]
        n_last = Yres.shape[1]
        Yh = torch.empty((B, n_last), dtype=torch.float32).pin_memory()
        single = len(layers) == 1 and not conv

        def host_step():
            if model is not None:  # model_infer drop-in: chunked H2D / graph chain / D2H
                model.infer_host_ptr(Xh.data_ptr(), Yh.data_ptr(), B, np.float32)
            elif conv and len(layers) == 1:  # host conv entry: image chunks, copies overlapped
                layers[0].conv_forward_host_ptr(Xh.data_ptr(), conv["N"], conv["H"], conv["W"], conv["C"], conv["k"],
                                                conv["s"], Yh.data_ptr())
            elif single:
                layers[0].forward_host_ptr(Xh.data_ptr(), Yh.data_ptr(), B, np.float32)
            else:
                Xd = torch.empty_like(X)
                Xd.copy_(Xh, non_blocking=True)
                step(src=Xd)
                Yh.copy_(Yres, non_blocking=True)
                torch.cuda.current_stream().synchronize()
            return float(Yh[0, 0])  # the step's result read on the host

        t_w = time.perf_counter()
        for _ in range(2):
            host_step()
        # enough host-timed steps for >= ~0.5 s of wall clock (short steps are noisy)
        Ke = int(min(200, max(3, min(K, 10), 0.5 / max((time.perf_counter() - t_w) / 2, 1e-6))))
        if dist:
            ke = torch.tensor([Ke], device=f"cuda:{local}")
            dist.all_reduce(ke, op=dist.ReduceOp.MAX)
            Ke = int(ke.item())
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(Ke):
            host_step()
        dt = (time.perf_counter() - t0) / Ke
        te = torch.tensor([dt], device=f"cuda:{local}")
        if dist:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        dt = float(te.item())
        h2d = X.numel() * 4
        d2h = B * n_last * 4
        e2e = {"value": (B if out_sharded else ws * B) / dt, "unit": "samples/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": dt * 1e3, "steps": Ke,
               "timer": "host wall clock around H2D + forward + D2H + host read (public API)"}

    # ---- e2e through the reference-signature C++ drop-in (tools/dropin_bench):
    # lmkan_b200::lmkan_forward(const LmKanLayer&, const Matrix&, Matrix&), fp64
    # X / Y in pageable host memory, exactly what an existing caller of
    # lmkan::lmkan_forward (layer.hpp:108-134) runs after the namespace swap.
    e2e_dropin = None
    dropin_bin = os.path.join(ROOT, "tools", "dropin_bench")
    if (not args.no_e2e and len(cfg["layers"]) == 1 and not conv and not out_sharded
            and os.path.exists(dropin_bin)):
        n_in0, n_out0 = cfg["layers"][0]
        Kd = max(3, min(K, 10))
        r = subprocess.run([dropin_bin, str(n_in0), str(n_out0), str(G), str(B), str(Kd), "2", str(local)],
                           capture_output=True, text=True, timeout=900,
                           env={**os.environ, "LMKAN_B200_PRECISION": str(args.precision)})
        if r.returncode == 0:
            d = json.loads(r.stdout.strip().splitlines()[-1])
            td = torch.tensor([d["ms_per_step"]], device=f"cuda:{local}")
            if dist:
                dist.all_reduce(td, op=dist.ReduceOp.MAX)
            e2e_dropin = {"value": ws * B / (float(td.item()) / 1e3), "unit": "samples/s",
                          "h2d_bytes_per_step": d["h2d_bytes_per_step"], "d2h_bytes_per_step": d["d2h_bytes_per_step"],
                          "ms_per_step": float(td.item()), "steps": d["steps"],
                          "api": "lmkan_b200::lmkan_forward(const LmKanLayer&, const Matrix&, Matrix&): fp64 X/Y in "
                                 "pageable host memory (tools/dropin_bench.cpp)",
                          "timer": "host wall clock per call, Y on the host when it returns"}
        else:
            e2e_dropin = {"error": (r.stderr or r.stdout)[-300:]}

    if rank != 0:
        if peers is not None:
            peers.close()
        if dist:
            dist.destroy_process_group()
        return
    clocks = sampler.summary()
    peak, peak_src = load_peaks()
    balg_row = sum(b_alg(a, b) for a, b in cfg["layers"])
    if args.precision == 64:  # 8-byte coefficients and I/O
        balg_row = sum(2 * b_alg(a, b) for a, b in cfg["layers"])
    achieved = B * balg_row / (kernel_ms / 1e3) / 1e9
    plan = layers[0].plan(B)
    if conv and hasattr(layers[0], "conv_plan"):  # the conv call's own plan (pixel records, L1-capped ring)
        cp = layers[0].conv_plan(conv["N"], conv["H"], conv["W"], conv["C"], conv["k"], conv["s"])
        plan.update(nbuf=cp["nbuf"], rows_per_cta=cp["rows_per_cta"], pixel_records=cp["pixel_records"])
    cpu = None
    if not args.no_cpu_baseline and ws == 1 and args.precision == 32:
        if out_sharded:  # 146 GB fp64 table does not fit the host: time a 16-output slice, scale by cost ~ n_out
            n_in0 = cfg["layers"][0][0]
            sl = pkg.Layer.random(n_in0, n_out0, G, seed=1000, gamma=1.0, device=local, out_range=(0, 16))
            r = cpu_reference(dict(cfg, layers=[(n_in0, 16)]), [sl.read_table()], budget_s=10)
            scale = 16 / n_out0
            extra = f"; 16-output slice of the {n_out0}-output layer, samples/s scaled by 16/{n_out0} (cost is linear in n_out)"
        else:
            tables = [lay.read_table() for lay in layers]
            r = cpu_reference(cfg, tables)
            scale, extra = 1.0, ""
        med = statistics.median(r["step_times"])
        cpu = {"value": r["rows"] / med * scale, "unit": "samples/s", "cores": r["cores"], "kind": r["kind"],
               "sample": f"{r['rows']} rows x {len(r['step_times'])} timed runs (median, {r['warmup']} warm-up) "
                         f"of the {cfg['name']} workload" + extra,
               "cpu_model": host_cpu_model(), "threads_env": "LMKAN_THREADS=nproc"}
    fmas = B * sum(fma_per_row(a, b) for a, b in cfg["layers"])
    out = {
        "metric": METRIC,
        "value": value,
        "unit": "samples/s",
        "n_gpus": ws,
        "steps": K,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": "strong" if out_sharded else "weak",
        "vs_baseline": None,
        "dtype": "fp64" if args.precision == 64 else "fp32",
        "precision": ("reference (fp64 table and accumulation, bit-identical to the reference forward)"
                      if args.precision == 64 else "fp32 gather (|y - y_ref| <= 1e-5 max(1, |y_ref|))"),
        "data": "synthetic: X ~ N(0,1) (torch CUDA generator), table ~ N(0, 1/pairs) from a device counter RNG",
        "config": config_dict(CONFIGS[args.config], ws, rank, shards, args.gather),
        "kernel_plan": dict(plan, n_out_local=cfg["layers"][0][1]),
        "l2_policy": (("inputs larger than L2: X %.0f MB, tables %.0f MB, outputs %.0f MB vs 126 MB L2; steps back to back"
                       if flush is None else
                       "L2 flushed between timed steps (256 MB write, outside each step's events): X %.0f MB, "
                       "tables %.0f MB, outputs %.0f MB fit the 126 MB L2") % (
            X.numel() * 4 / 1e6, sum(l.table_bytes for l in layers) / 1e6, sum(a.numel() * 4 for a in acts) / 1e6)),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": load_traffic(args.config),
                     "peak_source": peak_src, "kernel": "fwd_fused_kernel (gather; staged mode: K2)",
                     "alg_bytes_per_launch": B * balg_row, "kernel_ms": kernel_ms,
                     "kernel_share_of_step": kernel_ms / ms_per_step,
                     "note": "B_alg = 8*n_in*n_out + 4*(n_in+n_out) per row (gather-from-HBM model); "
                             "frac > 1 means table reuse from SMEM/L2",
                     "kernel_timing": ("CUDA events around each gather kernel on the launch stream, eager pass of "
                                       "the same K steps after the graph-replayed timed region")
                     if model is not None else
                     "CUDA events around each gather kernel on the launch stream, inside the timed region",
                     "fp32_fma_tflops": fmas / (kernel_ms / 1e3) / 1e12,
                     # the ceiling that binds the gather: one 4-byte
                     # coefficient per FMA through the 128 B/clk/SM shared-memory port
                     "smem_gather_ceiling": smem_ceiling(fmas / B * (2 if args.precision == 64 else 1),
                                                         clocks.get("sm_mhz"), kernel_ms, B),
                     # the same numerator against every level: > 1 means the
                     # level is not binding (reuse above it); the SMEM frac is the binding one
                     "levels": roofline_levels(achieved, fmas / (kernel_ms / 1e3), peak, clocks.get("sm_mhz"))},
        "clocks": clocks,
        "e2e": e2e,
        "e2e_dropin": e2e_dropin,
        "cpu_baseline": cpu,
        "gpu_launches": K * launches_per_step,
        "impl": "b200",
    }
    print(json.dumps(out))
    if peers is not None:
        peers.close()
    if dist:
        dist.destroy_process_group()


def reference_arm(args, cfg, ws):
    """bench.py --impl reference: the reference's own CPU lmkan_forward
    (oracle/_ref) on this host's cores, same workload, metric and config
    dict as the b200 arm. One step = one lmkan_forward pass over a bounded row
    sample of the workload (sized so W + K steps take about 90 s); exactly W
    untimed and K timed steps; ms_per_step / value are those of the sample
    rows actually run (value = sample rows / median step time)."""
    import numpy as np
    G = cfg["G"]
    rng = np.random.default_rng(1000)
    scale, run_cfg, extra = 1.0, cfg, ""
    if cfg.get("out_sharded"):  # the fp64 table (292 GB) does not fit the host: 16-output slice, scaled
        n_in0, n_out0 = cfg["layers"][0]
        run_cfg = dict(cfg, layers=[(n_in0, 16)])
        scale = 16 / n_out0
        extra = f"; 16-output slice, samples/s scaled by {scale:g} (cost is linear in n_out)"
    tables = [(rng.standard_normal(((G + 1) ** 2 * (a // 2) * b)).astype(np.float32).astype(np.float64)
               / np.sqrt(a // 2)).reshape(G + 1, G + 1, a // 2, b) for a, b in run_cfg["layers"]]
    step_s = max(0.05, min(3.0, 90.0 / (args.steps + args.warmup)))
    r = cpu_reference(run_cfg, tables, step_s=step_s, steps=args.steps, warmup=args.warmup)
    med = statistics.median(r["step_times"])
    v = r["rows"] / med * scale
    sample = (f"each step: lmkan_forward over {r['rows']} of the workload's {cfg['batch']} rows "
              f"({args.warmup} warm-up + {args.steps} timed steps, median){extra}")
    shards = (args.shards or ws) if cfg.get("out_sharded") else 1
    out = {
        "metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": med * 1e3, "higher_is_better": True,
        "scaling": "strong" if cfg.get("out_sharded") else "weak", "vs_baseline": None, "dtype": "fp64",
        "data": "synthetic: X ~ N(0,1), table ~ N(0, 1/pairs), fp32-representable values widened to fp64",
        "config": config_dict(cfg, ws, 0, shards, args.gather),
        "impl": "reference",
        "rows_per_step": r["rows"],
        "cpu_baseline": {"value": v, "unit": "samples/s", "cores": r["cores"], "kind": r["kind"], "sample": sample,
                         "cpu_model": host_cpu_model(), "threads_env": "LMKAN_THREADS=nproc"},
        "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
