"""Per-conv kernel times (CUDA events around each conv launch) of the AlexNet stack at
batch 128: protected forward vs unprotected, averaged over 10 forwards.  Env knobs
(FTC_NO_FUSED, FTC_TC_DEBUG bits) select experiment variants."""
import ctypes as C
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2003_12203_b200 import _abi, nets

lib = _abi.lib()
net = nets.alexnet()
dev = torch.device("cuda")
pn = nets.ProtectedNet(net, 128, 11, dev, nets.calibrate_taus(net, 128, 11, dev))
pn.set_input(torch.from_numpy(nets.net_input(net, 128, 3)).cuda())
for _ in range(3):
    pn.forward()
    pn.unprotected()
torch.cuda.synchronize()
res = {}
for mode in ("protected", "unprotected"):
    for L in pn.layers.values():
        lib.ftc_layer_set_timing(L.h, 1)
        lib.ftc_layer_kernel_time(L.h, None, None, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        if mode == "protected":
            pn.forward()
        else:
            pn.unprotected()
    e1.record()
    torch.cuda.synchronize()
    step = e0.elapsed_time(e1) / 10
    row = []
    for name, L in pn.layers.items():
        ms, n = C.c_double(), C.c_int32()
        lib.ftc_layer_kernel_time(L.h, C.byref(ms), C.byref(n), 1)
        lib.ftc_layer_set_timing(L.h, 0)
        row.append(f"{name}={ms.value / max(n.value, 1) * 1e3:.0f}")
    print(f"{os.environ.get('TAG', ''):12s} {mode:11s} step={step * 1e3:.0f}us conv_us: " + " ".join(row))
