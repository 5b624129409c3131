"""Small forwards through every kernel family, for compute-sanitizer runs
(memcheck / racecheck / synccheck): staged, fused, global, slabbed, narrow,
small-batch warps, duplicated-node tables, global node offsets, conv, model
chain, backward, multi-destination epilogue."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_07103_b200 as pkg  # noqa: E402


def run(env, n_in, n_out, G, rows):
    for k in [k for k in os.environ if k.startswith("LMKAN_B200_")]:
        del os.environ[k]
    os.environ.update(env)
    lay = pkg.Layer.random(n_in, n_out, G, seed=1)
    X = torch.randn((rows, n_in), device="cuda")
    Y = lay.forward(X)
    torch.cuda.synchronize()
    print(env, n_in, n_out, G, rows, float(Y.abs().sum()), flush=True)


run({}, 64, 64, 8, 1024)
run({}, 256, 192, 16, 1500)
run({"LMKAN_B200_MODE": "fused"}, 40, 72, 12, 1300)
run({"LMKAN_B200_MODE": "staged", "LMKAN_B200_SLABS": "2"}, 40, 72, 28, 700)
run({"LMKAN_B200_MODE": "global"}, 40, 72, 12, 300)
run({"LMKAN_B200_NW": "2", "LMKAN_B200_RT": "4"}, 64, 64, 8, 100)
run({}, 128, 1, 28, 3000)
run({}, 40, 16, 16, 3000)  # OT = 16 duplicated-node table (fused)
run({"LMKAN_B200_MODE": "staged"}, 40, 16, 16, 3000)  # DUP, staged
run({}, 128, 128, 28, 40000)  # staged 1024-row tile with node offsets from global (GOFF)
run({}, 12, 128, 28, 2000)
lay = pkg.Layer.random(144, 16, 16, seed=2)
img = torch.randn((3, 10, 10, 16), device="cuda")
print("conv", float(lay.conv_forward(img, 3, 1).abs().sum()))
m = pkg.Model.from_layers([pkg.Layer.random(12, 32, 8, seed=3), pkg.Layer.random(32, 2, 8, seed=4)])
st = torch.cuda.Stream()
Xm = torch.randn((500, 12), device="cuda")
Ym = torch.empty((500, 2), device="cuda")
for _ in range(2):
    m.infer_into(Xm, Ym, st)
st.synchronize()
print("model", float(Ym.abs().sum()))
P = np.random.default_rng(0).standard_normal((9, 9, 3, 5))
bl = pkg.Layer.from_host(6, 5, 8, P, 0.7)
dP, dX = bl.backward(torch.from_numpy(P).cuda(), torch.randn((200, 6), device="cuda", dtype=torch.float64),
                     torch.randn((200, 5), device="cuda", dtype=torch.float64))
print("backward", float(dP.abs().sum()), float(dX.abs().sum()))
sl = pkg.Layer.random(64, 48, 8, seed=5, out_range=(16, 32))
bufs = [torch.zeros((300, 48), device="cuda") for _ in range(3)]
sl.forward_dests(torch.randn((300, 64), device="cuda"), [b.data_ptr() for b in bufs], 48, 16)
torch.cuda.synchronize()
print("dests", float(bufs[2].abs().sum()))
# round 2: half-swapped plain OT = 16 sheets (staged + fused), pair-block
# summation, narrow pair blocks, pixel-record conv, reference precision (every
# sheet width and the L2-sheet variant), production-record dumps, large grids,
# pageable host staging
run({}, 64, 16, 28, 2000)                               # plain OT 16, half swap, staged
run({"LMKAN_B200_MODE": "fused"}, 64, 16, 28, 2000)     # half swap, in-kernel locate
run({"LMKAN_B200_PAIR_BLOCK": "4"}, 40, 24, 8, 900)     # pair blocks (fold into Y)
run({"LMKAN_B200_PAIR_BLOCK": "4"}, 46, 3, 8, 700)      # narrow kernel pair blocks
run({}, 10, 7, 100, 300)                                # G = 100: global-sheet mode
lay = pkg.Layer.random(9 * 32, 32, 16, seed=7)
print("conv pixel", float(lay.conv_forward(torch.randn((2, 12, 12, 32), device="cuda"), 3, 1).abs().sum()))
for n_in, n_out, G in [(64, 64, 8), (30, 40, 28), (12, 9, 40), (6, 3, 200)]:
    Pe = np.random.default_rng(G).standard_normal((G + 1, G + 1, n_in // 2, n_out))
    le = pkg.Layer.from_host(n_in, n_out, G, Pe, 0.9, precision=64)
    Ye = le.forward(torch.randn((700, n_in), device="cuda", dtype=torch.float64))
    torch.cuda.synchronize()
    print("exact", G, float(Ye.abs().sum()))
lr = pkg.Layer.random(64, 16, 28, seed=8)
Xr = torch.randn((600, 64), device="cuda")
for v in ("k1", "k1_smem", "in_kernel"):
    i1, i2, ag = lr.records(Xr, v)
torch.cuda.synchronize()
print("records", int(i1.sum()), int(i2.sum()))
lh = pkg.Layer.random(96, 80, 12, seed=9)
print("host staging", float(np.abs(lh.forward_host(np.random.default_rng(1).standard_normal((20000, 96)))).sum()))
# round 2, late: CTA-order groups (cta_tile, incl. the pair-block fold's
# re-derived tile) and the pixel-record conv with its L1-capped ring
run({"LMKAN_B200_CTA_GROUP": "2"}, 256, 192, 16, 1500)
run({"LMKAN_B200_CTA_GROUP": "3", "LMKAN_B200_PAIR_BLOCK": "4"}, 40, 80, 12, 900)
lay = pkg.Layer.random(9 * 32, 32, 16, seed=7)
print("conv stage 2", float(lay.conv_forward(torch.randn((256, 18, 18, 32), device="cuda"), 3, 1).abs().sum()))
