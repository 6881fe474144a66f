"""Quick tcgen05-engine check against the SIMT engine and the oracle (dev tool)."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
import paper_2003_12203_b200 as F
from paper_2003_12203_b200 import synth
import oracle_py as O

def run(N, C, H, M, R, stride=1, pad=1, bias=False, seed=0, timeit=False):
    p = F.ConvParams(stride=stride, pad=pad, bias_enabled=bias)
    D = synth.relu_like((N, C, H, H), seed)
    W = synth.he_normal(M, C, R, seed + 1)
    B = synth.uniform((M,), -0.1, 0.1, seed + 2) if bias else None
    L = F.ProtectedConv(W, B, p, N, H)
    Dg = torch.from_numpy(D).cuda()
    F.set_conv_engine("tc"); Ot = L.conv_forward(Dg); torch.cuda.synchronize()
    Ot = Ot.cpu().numpy()
    Oo = O.conv_f32(O.dims(N, C, H, M, R, stride, pad, 1, bias), D, W, B)
    e = np.abs(Ot - Oo) / np.maximum(1, np.maximum(np.abs(Ot), np.abs(Oo)))
    msg = f"N={N} C={C} H={H} M={M} R={R} s={stride} p={pad}: tc err {e.max():.3e}"
    if timeit:
        O_ = torch.empty(L.out_shape, device="cuda")
        for _ in range(3): L.conv_forward(Dg, O_)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); n = 20
        for _ in range(n): L.conv_forward(Dg, O_)
        e1.record(); e1.synchronize(); ms = e0.elapsed_time(e1) / n
        E = L.E; fl = 2.0 * N * M * E * E * C * R * R
        msg += f"  {ms*1e3:.1f} us  {fl/ms/1e9:.1f} TFLOP/s"
    print(msg, flush=True)
    L.close()
    return e.max()

worst = 0
for cfg in [(2, 32, 8, 32, 3), (16, 64, 56, 64, 3, 1, 1, False, 0, True), (3, 3, 31, 96, 11, 4, 0),
            (4, 96, 27, 256, 5, 1, 2), (2, 256, 13, 384, 3), (1, 20, 9, 40, 1, 1, 0),
            (5, 7, 10, 425, 3, 1, 1, True), (2, 1024, 13, 128, 3, 1, 1), (128, 256, 13, 384, 3, 1, 1, False, 3, True),
            (128, 96, 27, 256, 5, 1, 2, False, 4, True)]:
    worst = max(worst, run(*cfg))
print("WORST", worst)
