"""In-net vs alone, protected (FUSE) vs plain conv kernel durations (run under ncu): the
VGG-19 net protected, then unprotected, then c3/c4/c6 alone protected on the net's
activations."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2003_12203_b200 as F
from paper_2003_12203_b200 import nets, synth
dev = torch.device("cuda:0")
net = nets.vgg19()
pn = nets.ProtectedNet(net, 64, 11, dev)
pn.set_input(nets.net_input(net, 64, 1000))
pn.forward()
torch.cuda.synchronize()
print("net protected done", flush=True)
pn.unprotected()
torch.cuda.synchronize()
print("net unprotected done", flush=True)
plan = F.LayerPlan(rc_enabled=True, clc_enabled=True, tau=1e-2)
for op, Cin, H, E in pn.convs:
    if op.dst not in os.environ.get("LAYERS", "c3,c4,c6").split(","):
        continue
    W, b = pn.weights[op.dst]
    L = F.ProtectedConv(W, b, F.ConvParams(stride=op.stride, pad=op.pad, bias_enabled=op.bias), 64, H)
    Dr = pn.buf[op.src].clone()
    for _ in range(2):
        O, rep = L.protected(Dr, plan)
    print(op.dst, "alone protected", rep.detected, flush=True)
    L.close()
