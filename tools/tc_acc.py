"""TC conv accuracy vs FP64 (and the reference-order FP32 loop) on net-like shapes."""
import sys
import numpy as np
import torch
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
import paper_2003_12203_b200 as F
from paper_2003_12203_b200 import synth
import oracle_py as O
rel = lambda a, b: np.abs(a - b) / np.maximum(1, np.maximum(np.abs(a), np.abs(b)))
out = []
for (N, C, H, M, R, pad) in [(4, 96, 27, 256, 5, 2), (4, 64, 56, 64, 3, 1), (2, 256, 13, 384, 3, 1), (2, 512, 14, 512, 3, 1)]:
    D = synth.relu_like((N, C, H, H), 0); W = synth.he_normal(M, C, R, 1)
    L = F.ProtectedConv(W, None, F.ConvParams(pad=pad), N, H)
    Og = L.conv_forward(torch.from_numpy(D).cuda()).cpu().numpy()
    d = O.dims(N, C, H, M, R, 1, pad, 1, False)
    O64 = O.conv_f64(d, D.astype(np.float64), W.astype(np.float64), None)
    Or = O.conv_f32(d, D, W, None)
    out.append(f"K={C*R*R}: tc {rel(Og, O64).max():.2e} ref {rel(Or, O64).max():.2e}")
    L.close()
print(" | ".join(out))
