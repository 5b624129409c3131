import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2509_07103_b200 as pkg
lay = pkg.Layer.random(128, 128, 16, seed=1)
print(lay.plan(40000))
X = torch.randn((40000, 128), device="cuda")
Y = lay.forward(X); torch.cuda.synchronize(); print(float(Y.abs().sum()))
