"""Run-to-run determinism of the tcgen05 conv: the same layer on the same input, many
times; every output must be bitwise equal to the first (r02 investigation)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2003_12203_b200 as F
from paper_2003_12203_b200 import synth

shapes = [("vgg_c7", 64, 256, 56, 256, 3, 1), ("alex_c3", 128, 256, 13, 384, 3, 1), ("vgg_c2", 64, 64, 224, 64, 3, 1),
          ("vgg_c12", 64, 512, 28, 512, 3, 1)]
reps = int(os.environ.get("DET_REPS", "120"))
for name, N, C, H, M, R, p in shapes:
    D = torch.from_numpy(synth.relu_like((N, C, H, H), 1)).cuda()
    W = synth.he_normal(M, C, R, 2)
    L = F.ProtectedConv(W, None, F.ConvParams(pad=p), N, H)
    plan = F.LayerPlan(rc_enabled=True, clc_enabled=True, tau=0.1)
    for mode in ("conv", "protected"):
        ref = None
        bad = 0
        where = []
        for r in range(reps):
            if mode == "conv":
                O = L.conv_forward(D)
            else:
                O, rep = L.protected(D, plan)
            torch.cuda.synchronize()
            if ref is None:
                ref = O.clone()
                continue
            d = (O.view(torch.int32) != ref.view(torch.int32))
            if d.any():
                bad += 1
                idx = d.nonzero()[:4].tolist()
                where.append((r, int(d.sum()), idx))
        print(f"{name} {mode}: {bad}/{reps - 1} runs differ", where[:4], flush=True)
    L.close()
