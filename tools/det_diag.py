"""Run-to-run determinism diagnosis (r02): the same protected layer on the same input,
many times; on a difference, report whether the staged NHWC input copy (the conv's A
operand source) differed too, and the ULP distance of the differing outputs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import torch
import paper_2003_12203_b200 as F
from paper_2003_12203_b200 import _abi, synth

shape = tuple(int(v) for v in os.environ.get("DET_SHAPE", "64,512,28,512,3,1").split(","))
reps = int(os.environ.get("DET_REPS", "200"))
mode = os.environ.get("DET_MODE", "protected")
N, Cc, H, M, R, pad = shape
D = torch.from_numpy(synth.relu_like((N, Cc, H, H), 1)).cuda()
W = synth.he_normal(M, Cc, R, 2)
L = F.ProtectedConv(W, None, F.ConvParams(pad=pad), N, H)
plan = F.LayerPlan(rc_enabled=True, clc_enabled=True, tau=0.1)
lib = _abi.lib()
p = C.c_void_p()
lib.ftc_layer_input_nhwc(L.h, C.byref(p))
Dt = torch.empty((N * H * H * Cc,), device="cuda")
O = torch.empty(L.out_shape, device="cuda")


def run():
    global O
    if mode == "conv":
        L.conv_forward(D, O)
        det = False
    else:
        O, rep = L.protected(D, plan)
        det = rep.detected
    torch.cuda.synchronize()
    if p.value:
        lib.ftc_memcpy(C.c_void_p(Dt.data_ptr()), p, Dt.numel() * 4, 2, None)
    return O.clone(), Dt.clone(), det


O0, Dt0, _ = run()
nO = nD = ndet = 0
for r in range(reps):
    Ok, Dk, det = run()
    ndet += int(det)
    dO = (Ok.view(torch.int32) != O0.view(torch.int32))
    dD = (Dk.view(torch.int32) != Dt0.view(torch.int32))
    if dO.any() or dD.any():
        nO += int(dO.any().item())
        nD += int(dD.any().item())
        idx = dO.nonzero()[:4].tolist()
        ulps = [int(Ok[tuple(i)].view(torch.int32)) - int(O0[tuple(i)].view(torch.int32)) for i in idx]
        didx = dD.nonzero()[:4].flatten().tolist()
        print(f"run {r}: O diff {int(dO.sum())} at {idx} ulps {ulps}; Dt diff {int(dD.sum())} at {didx}", flush=True)
print(f"{shape} {mode} pdl={'off' if os.environ.get('FTC_NO_PDL') else 'on'}: O differs in {nO}/{reps}, "
      f"Dt differs in {nD}/{reps}, detections {ndet}")
