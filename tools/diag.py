import sys
import numpy as np
import torch
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
import paper_2003_12203_b200 as F
from paper_2003_12203_b200 import synth, nets
import oracle_py as O

# (1) verdict scenario of tests/cpp/test_api.cpp
D = O.tensor_random((3, 8, 10, 10), 500); W = O.tensor_random((6, 8, 3, 3), 501)
p = F.ConvParams(pad=1)
for eng in ("simt", "tc"):
    F.set_conv_engine(eng)
    L = F.ProtectedConv(W, None, p, 3, 10)
    Dg = torch.from_numpy(D).cuda()
    Oc = L.conv_forward(Dg).cpu().numpy()
    plan = F.LayerPlan(rc_enabled=True, clc_enabled=True, tau=1e-5)
    f = F.Fault("output", 1, 2, 3, 4, "add", value=9.0)
    Og, rep = L.protected(Dg, plan, [f])
    Of = Oc.copy(); Of[1, 2, 3, 4] = np.float32(Of[1, 2, 3, 4] + np.float32(9.0))
    ref = O.protected_layer(O.dims(3, 8, 10, 6, 3, 1, 1), D, W, None, True, True, 1e-5, O_conv=Of)
    print(eng, "gpu:", rep.verdict(), rep.n_flagged, rep.max_rel_dev)
    print(eng, "ref:", {k: ref[k] for k in ("detected", "stage", "stages_attempted", "corrected_blocks")})
    Oh, reph = L.protected_host(D, plan, [f])
    print(eng, "host:", reph.verdict())
    L.close()
F.set_conv_engine("tc")

# (2) error budget of AlexNet c2 on real activations: GPU and reference vs FP64
net = nets.alexnet()
pn = nets.ProtectedNet(net, 4, 11, torch.device("cuda"))
pn.set_input(torch.from_numpy(nets.net_input(net, 4, 3)).cuda())
pn.unprotected(); torch.cuda.synchronize()
for name in ("c1", "c2", "c3", "c5"):
    op, Cin, H, E = [c for c in pn.convs if c[0].dst == name][0]
    Dn = pn.buf[op.src].cpu().numpy(); Og = pn.buf[op.dst].cpu().numpy()
    Wn, b = pn.weights[name]
    d = O.dims(4, Cin, H, op.M, op.R, op.stride, op.pad, 1, op.bias)
    Or = O.conv_f32(d, Dn, Wn, b); O64 = O.conv_f64(d, Dn.astype(np.float64), Wn.astype(np.float64), None if b is None else b.astype(np.float64))
    m = lambda a, b_: (np.abs(a - b_) / np.maximum(1, np.maximum(np.abs(a), np.abs(b_)))).max()
    print(name, f"|O|max {np.abs(O64).max():.2f}  gpu-vs-f64 {m(Og, O64):.2e}  ref-vs-f64 {m(Or, O64):.2e}  gpu-vs-ref {m(Og, Or):.2e}")
