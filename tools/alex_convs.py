"""Profiling target: the AlexNet conv stack (batch 128) protected forward, after warm-up.
Each forward launches the 5 k_conv_tc kernels once (ncu: -k regex:k_conv_tc -s 10 -c 5)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2003_12203_b200 import nets
net = nets.alexnet()
dev = torch.device("cuda")
pn = nets.ProtectedNet(net, 128, 11, dev, nets.calibrate_taus(net, 128, 11, dev))
pn.set_input(torch.from_numpy(nets.net_input(net, 128, 3)).cuda())
for _ in range(8):
    pn.forward()
torch.cuda.synchronize()
print("ok")
