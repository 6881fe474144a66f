import sys
import numpy as np
import torch
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
import paper_2003_12203_b200 as F
from paper_2003_12203_b200 import nets
import oracle_py as O
net = nets.resnet18()
pn = nets.ProtectedNet(net, 2, 11, torch.device("cuda"))
pn.set_input(torch.from_numpy(nets.net_input(net, 2, 3)).cuda())
pn.unprotected(); torch.cuda.synchronize()
for name in ("b3_proj", "b3_c1", "b5_proj", "stem"):
    op, Cin, H, E = [c for c in pn.convs if c[0].dst == name][0]
    Dn = pn.buf[op.src].cpu().numpy(); Og = pn.buf[op.dst].cpu().numpy()
    Wn, b = pn.weights[name]
    d = O.dims(2, Cin, H, op.M, op.R, op.stride, op.pad, 1, op.bias)
    Or = O.conv_f32(d, Dn, Wn, b)
    O64 = O.conv_f64(d, Dn.astype(np.float64), Wn.astype(np.float64), None if b is None else b.astype(np.float64))
    F.set_conv_engine("simt"); Os = pn.layers[name].conv_forward(pn.buf[op.src]).cpu().numpy(); F.set_conv_engine("tc")
    rel = lambda a, b_: np.abs(a - b_) / np.maximum(1, np.maximum(np.abs(a), np.abs(b_)))
    for lab, X in (("tc", Og), ("simt", Os), ("ref", Or)):
        e = rel(X, O64); i = np.unravel_index(np.argmax(e), e.shape)
        print(name, lab, f"max {e.max():.2e} at {i} val {O64[i]:.5f} got {X[i]:.7f} absmax|O| {np.abs(O64).max():.2f}")
    # per-term magnitude of the worst element
    print("  D range", Dn.min(), Dn.max(), "W absmax", np.abs(Wn).max(), "K", Cin * op.R * op.R)
