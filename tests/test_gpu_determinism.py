"""Run-to-run determinism of the tcgen05 conv (repaired planes must be bitwise the
fault-free output, and a replayed layer must reproduce its first run): the same layer
on the same input, many times, every output bitwise equal to the first.  Shapes cover
the BN = 64 / 128 tiles, the TMA im2col and register-gather engines and a long K."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SHAPES = [  # N, C, H, M, R, pad
    (16, 64, 56, 64, 3, 1),     # config 1 (BN 64, TMA im2col)
    (32, 256, 28, 256, 3, 1),   # VGG-like (BN 128, K = 2304)
    (16, 3, 67, 96, 11, 0),     # C = 3 stem (register gather)
    (32, 512, 14, 512, 3, 1),   # K = 4608
]


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_conv_bitwise_repeatable(shape):
    import torch
    import paper_2003_12203_b200 as F
    from paper_2003_12203_b200 import synth
    N, C, H, M, R, pad = shape
    D = torch.from_numpy(synth.relu_like((N, C, H, H), 1)).cuda()
    W = synth.he_normal(M, C, R, 2)
    L = F.ProtectedConv(W, None, F.ConvParams(pad=pad), N, H)
    plan = F.LayerPlan(rc_enabled=True, clc_enabled=True, tau=0.1)
    O = torch.empty(L.out_shape, device="cuda")
    L.conv_forward(D, O)
    ref = O.clone()
    bad = 0
    for r in range(40):
        if r % 2:
            L.conv_forward(D, O)
        else:
            O, rep = L.protected(D, plan)
            assert not rep.detected
        torch.cuda.synchronize()
        bad += int((O.view(torch.int32) != ref.view(torch.int32)).any().item())
    L.close()
    assert bad == 0, f"{bad}/40 runs differ from the first"
