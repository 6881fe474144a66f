"""Run the config-1 (or AlexNet conv2) conv a few times (profiling target)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2003_12203_b200 as F
from paper_2003_12203_b200 import synth
which = sys.argv[1] if len(sys.argv) > 1 else "c1"
if which == "c1":
    N, C, H, M, R, pad = 16, 64, 56, 64, 3, 1
else:
    N, C, H, M, R, pad = 128, 96, 27, 256, 5, 2
D = synth.relu_like((N, C, H, H), 0); W = synth.he_normal(M, C, R, 1)
L = F.ProtectedConv(W, None, F.ConvParams(pad=pad), N, H)
Dg = torch.from_numpy(D).cuda(); O = torch.empty(L.out_shape, device="cuda")
for _ in range(4): L.conv_forward(Dg, O)
torch.cuda.synchronize(); print("ok")
