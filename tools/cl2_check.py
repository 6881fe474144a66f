"""CTA-pair conv (FTC_TC_CL=2) against the single-CTA kernel: bitwise-equal outputs
(unprotected and protected, odd and even tile counts) -- run once with FTC_TC_CL unset to
write the outputs, once with FTC_TC_CL=2 to compare."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2003_12203_b200 as F
from paper_2003_12203_b200 import synth

shapes = [(64, 256, 56, 256, 3, 1), (37, 64, 57, 64, 3, 1), (64, 128, 28, 320, 3, 1), (33, 512, 14, 512, 3, 1),
          (50, 64, 31, 128, 1, 0)]
mode = os.environ.get("FTC_TC_CL", "0")
out = os.environ.get("CL2_DIR", "/tmp/cl2")
os.makedirs(out, exist_ok=True)
bad = 0
for i, (N, C, H, M, R, pad) in enumerate(shapes):
    D = torch.from_numpy(synth.relu_like((N, C, H, H), 10 + i)).cuda()
    W = synth.he_normal(M, C, R, 20 + i)
    B = synth.uniform((M,), -0.1, 0.1, 30 + i)
    L = F.ProtectedConv(W, B, F.ConvParams(pad=pad, bias_enabled=True), N, H)
    O1 = L.conv_forward(D).cpu().numpy()
    O2, rep = L.protected(D, F.LayerPlan(rc_enabled=True, clc_enabled=True, tau=1e-3))
    O2 = O2.cpu().numpy()
    assert not rep.detected, rep
    f = os.path.join(out, f"o{i}.npy")
    if mode == "2":
        ref = np.load(f)
        same1 = np.array_equal(ref, O1)
        same2 = np.array_equal(ref, O2)
        print(f"shape {i} {(N, C, H, M, R, pad)}: conv bitwise {same1}, protected bitwise {same2}", flush=True)
        bad += (not same1) + (not same2)
    else:
        assert np.array_equal(O1, O2)
        np.save(f, O1)
        print(f"shape {i}: saved", flush=True)
    L.close()
print("CL2 CHECK", "FAIL" if bad else "OK")
