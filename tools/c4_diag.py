"""Why do VGG c3/c4 run slower inside the net than the same shapes alone?  Runs the VGG-19
net once, then the convs c3 / c4 / c6 alone on (A) the net's real activations, (B) seeded
relu_like inputs, (C) zeros -- run under ncu (gpu__time_duration) and read the k_conv_tc
launches in order."""
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
print("net done", flush=True)
for op, Cin, H, E in pn.convs:
    if op.dst not in os.environ.get("LAYERS", "c3,c4,c6").split(","):
        continue
    W, b = pn.weights[op.dst]
    L = F.ProtectedConv(W, b, F.ConvParams(stride=op.stride, pad=op.pad, bias_enabled=op.bias), 64, H)
    O = torch.empty(L.out_shape, device=dev)
    Dr = pn.buf[op.src].clone()
    Ds = torch.from_numpy(synth.relu_like((64, Cin, H, H), 5)).to(dev)
    Dz = torch.zeros_like(Dr)
    Dn = torch.randn_like(Dr)
    for tag, D in (("real", Dr), ("relu_like", Ds), ("zeros", Dz), ("randn", Dn)):
        print(op.dst, tag, "mean", float(D.mean()), "zeros", float((D == 0).float().mean()), "max", float(D.max()), flush=True)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        L.conv_forward(D, O)
        ev[0].record()
        for _ in range(3):
            L.conv_forward(D, O)
        ev[1].record()
        torch.cuda.synchronize()
        print("   call (transpose + conv) us:", ev[0].elapsed_time(ev[1]) / 3 * 1e3, flush=True)
    L.close()
