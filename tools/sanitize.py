"""Workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): small
protected layers on both tensor-core engines (register gather C=3/16, TMA im2col C=32),
the fused multi-layer clean path with its glue kernels (AlexNet-shaped stack at batch 2),
one faulted layer through the error path (CoC repair) and one RC pattern."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2003_12203_b200 as F
from paper_2003_12203_b200 import nets, synth

torch.cuda.set_device(0)
for N, C, H, M, R, pad in [(2, 3, 19, 32, 5, 2), (4, 16, 14, 24, 3, 1), (4, 32, 14, 40, 3, 1), (2, 64, 9, 128, 3, 1)]:
    D = torch.from_numpy(synth.relu_like((N, C, H, H), 1)).cuda()
    W = synth.he_normal(M, C, R, 2)
    L = F.ProtectedConv(W, None, F.ConvParams(pad=pad), N, H)
    plan = F.LayerPlan(rc_enabled=True, clc_enabled=True, tau=1e-3)
    O, rep = L.protected(D, plan)
    assert not rep.detected
    E = L.out_shape[-1]
    _, rep = L.protected(D, plan, [F.Fault("output", 1, 3, 1, 2, "add", value=5.0)])
    assert rep.stage == "coc", rep.stage
    _, rep = L.protected(D, plan, [F.Fault("output", 1, -1, 1, 2, "add", value=3.0, m_coef=0.01)])
    print(f"layer {N},{C},{H},{M},{R}: ok ({rep.stage})", flush=True)
    L.close()
net = nets.alexnet()
pn = nets.ProtectedNet(net, 2, 11, torch.device("cuda"))
pn.set_input(torch.from_numpy(nets.net_input(net, 2, 3)).cuda())
reps = pn.forward()
pn.unprotected()
torch.cuda.synchronize()
print("alexnet b2 stack:", {k: r.stage for k, r in reps.items()}, flush=True)
pn.close()
