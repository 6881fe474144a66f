import sys, torch
sys.path.insert(0, ".")
import paper_2003_12203_b200 as F
from paper_2003_12203_b200 import synth
import numpy as np
N, C, H, M, R, s = 128, 3, 227, 96, 11, 4
D = np.random.default_rng(0).standard_normal((N, C, H, H)).astype(np.float32); W = synth.he_normal(M, C, R, 1)
L = F.ProtectedConv(W, None, F.ConvParams(stride=s), N, H)
Dg = torch.from_numpy(D).cuda(); O = torch.empty(L.out_shape, device="cuda")
for _ in range(3): L.conv_forward(Dg, O)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): L.conv_forward(Dg, O)
e1.record(); e1.synchronize()
print(f"conv1 {e0.elapsed_time(e1) / 10 * 1e3:.1f} us")
