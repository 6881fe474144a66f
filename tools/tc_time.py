import sys, torch
sys.path.insert(0, ".")
import paper_2003_12203_b200 as F
from paper_2003_12203_b200 import synth
res = []
for (N, C, H, M, R, pad) in [(128, 96, 27, 256, 5, 2), (16, 64, 56, 64, 3, 1), (128, 256, 13, 384, 3, 1)]:
    D = synth.relu_like((N, C, H, H), 0); W = synth.he_normal(M, C, R, 1)
    L = F.ProtectedConv(W, None, F.ConvParams(pad=pad), N, H)
    Dg = torch.from_numpy(D).cuda(); O = torch.empty(L.out_shape, device="cuda")
    for _ in range(3): L.conv_forward(Dg, O)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): L.conv_forward(Dg, O)
    e1.record(); e1.synchronize()
    res.append(f"{e0.elapsed_time(e1) / 10 * 1e3:7.1f}us")
    L.close()
print(" ".join(res))
