"""Run-to-run determinism, detail: values and ULP distance of differing elements."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2003_12203_b200 as F
from paper_2003_12203_b200 import synth
N, C, H, M, R = 64, 256, 56, 256, 3
reps = int(os.environ.get("DET_REPS", "300"))
D = torch.from_numpy(synth.relu_like((N, C, H, H), 1)).cuda()
W = synth.he_normal(M, C, R, 2)
L = F.ProtectedConv(W, None, F.ConvParams(pad=1), N, H)
O = torch.empty(L.out_shape, device="cuda")
L.conv_forward(D, O); torch.cuda.synchronize()
ref = O.clone()
votes = {}
for r in range(reps):
    L.conv_forward(D, O)
    torch.cuda.synchronize()
    d = (O.view(torch.int32) != ref.view(torch.int32))
    if d.any():
        for idx in d.nonzero().tolist():
            a, b = float(O[tuple(idx)]), float(ref[tuple(idx)])
            ulp = int(O[tuple(idx)].view(torch.int32)) - int(ref[tuple(idx)].view(torch.int32))
            key = tuple(idx)
            votes.setdefault(key, []).append((r, a, b, ulp))
        print(f"run {r}: {int(d.sum())} elements differ", flush=True)
for k, v in votes.items():
    print("elem", k, "n_events", len(v), v[:4])
# majority value per element: is the REF the outlier?
