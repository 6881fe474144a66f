"""The Python API refuses tensors the C ABI would read or write out of bounds
(ADVICE r1): CPU / wrong dtype / non-contiguous / wrong shape -> ShapeError, before
any device pointer crosses the ABI (the reference raises ShapeError from
check_conv_shapes, conv.hpp:16-37)."""
import numpy as np
import pytest

import paper_2003_12203_b200 as F
from paper_2003_12203_b200 import synth

pytestmark = pytest.mark.gpu


def test_layer_entry_points_validate_tensors():
    import torch
    W = synth.he_normal(8, 4, 3, 1)
    L = F.ProtectedConv(W, None, F.ConvParams(pad=1), 2, 6)
    D = torch.from_numpy(synth.relu_like((2, 4, 6, 6), 2)).cuda()
    O = torch.empty((2, 8, 6, 6), device="cuda")
    plan = F.LayerPlan(rc_enabled=True, clc_enabled=True, tau=1e-3)
    bad_D = [D.cpu(), D.half(), D.double(), D.transpose(2, 3), D[:1], D.reshape(2, 4, 36)]
    for bD in bad_D:
        with pytest.raises(F.ShapeError):
            L.conv_forward(bD, O)
        with pytest.raises(F.ShapeError):
            L.protected(bD, plan, O=O)
        with pytest.raises(F.ShapeError):
            L.launch(bD, O, plan)
    for bO in [O.cpu(), O[:, :4], torch.empty((2, 8, 6, 5), device="cuda"), O.transpose(2, 3)]:
        with pytest.raises(F.ShapeError):
            L.conv_forward(D, bO)
        with pytest.raises(F.ShapeError):
            L.check(D, bO, plan)
    cd = torch.zeros((4, 6, 6), dtype=torch.float32, device="cuda")
    with pytest.raises(F.ShapeError):
        L.launch_cd1(D, O, cd, plan)  # float32 workspace
    with pytest.raises(F.ShapeError):
        L.launch_ck(D, O, cd.double(), cd, plan)
    # the valid call still works after the refusals
    Og, rep = L.protected(D, plan)
    torch.cuda.synchronize()
    assert not rep.detected and Og.shape == (2, 8, 6, 6)
    L.close()
