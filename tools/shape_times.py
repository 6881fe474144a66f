"""Conv kernel time (CUDA events around the conv launch, layer timing hook) for a list of
layer shapes: the VGG-19 / ResNet-18 / config-1 shapes that run BN = 64 tiles and the
3x3 BN = 128 ones.  SHAPES env: 'N,C,H,M,R,pad[,stride];...'."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import torch
import paper_2003_12203_b200 as F
from paper_2003_12203_b200 import _abi, synth
default = "16,64,56,64,3,1;64,64,224,64,3,1;64,128,112,128,3,1;64,256,56,256,3,1;64,512,28,512,3,1;256,64,56,64,3,1;128,96,27,256,5,2"
lib = _abi.lib()
for spec in os.environ.get("SHAPES", default).split(";"):
    v = [int(x) for x in spec.split(",")]
    N, Cc, H, M, R, pad = v[:6]
    U = v[6] if len(v) > 6 else 1
    D = torch.from_numpy(synth.relu_like((N, Cc, H, H), 1)).cuda()
    W = synth.he_normal(M, Cc, R, 2)
    L = F.ProtectedConv(W, None, F.ConvParams(pad=pad, stride=U), N, H)
    O = torch.empty(L.out_shape, device="cuda")
    for _ in range(3):
        L.conv_forward(D, O)
    torch.cuda.synchronize()
    lib.ftc_layer_set_timing(L.h, 1)
    lib.ftc_layer_kernel_time(L.h, None, None, 1)
    for _ in range(10):
        L.conv_forward(D, O)
    torch.cuda.synchronize()
    ms = C.c_double()
    n = C.c_int32()
    lib.ftc_layer_kernel_time(L.h, C.byref(ms), C.byref(n), 1)
    E = L.out_shape[-1]
    us = ms.value / n.value * 1e3
    fl = 2.0 * N * M * E * E * Cc * R * R
    print(f"{spec:24s} {us:9.1f} us  {fl / us / 1e6:7.1f} TFLOP/s", flush=True)
    L.close()
