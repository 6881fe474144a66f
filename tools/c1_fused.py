"""config1 protected launch time (events) under FTC_TC_DEBUG variants (fused-detect parts)."""
import sys, torch
sys.path.insert(0, ".")
import paper_2003_12203_b200 as F
from paper_2003_12203_b200 import synth
N, C, H, M, R, pad = 16, 64, 56, 64, 3, 1
D = synth.relu_like((N, C, H, H), 0); W = synth.he_normal(M, C, R, 1)
L = F.ProtectedConv(W, None, F.ConvParams(pad=pad), N, H)
Dg = torch.from_numpy(D).cuda(); O = torch.empty(L.out_shape, device="cuda")
plan = F.LayerPlan(tau=1e-3)
for _ in range(5):
    L.launch(Dg, O, plan); L.finish()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
t = 0.0
for _ in range(20):
    e0.record(); L.launch(Dg, O, plan); e1.record(); L.finish(); t += e0.elapsed_time(e1)
u = 0.0
for _ in range(20):
    e0.record(); L.conv_forward(Dg, O); e1.record(); e1.synchronize(); u += e0.elapsed_time(e1)
print(f"protected {t / 20 * 1e3:.1f} us   conv_forward {u / 20 * 1e3:.1f} us")
