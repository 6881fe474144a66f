"""GPU tests of the engine paths added for speed: TMA im2col geometry, the act+pool glue
that stages the next layer's NHWC copy, the staging guard, and the opt-in fused
clean-path CoC-D (verdict parity with run_protected_layer<double>)."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle_py as O
from conftest import ROOT


def _rel(a, b):
    return np.abs(a - b) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))


@pytest.mark.gpu
@pytest.mark.parametrize("N,C,H,M,R,s,p", [(2, 32, 15, 40, 3, 2, 1), (3, 64, 9, 24, 1, 1, 0), (2, 32, 11, 70, 5, 1, 2),
                                           (2, 96, 13, 130, 3, 1, 1), (1, 32, 17, 32, 3, 2, 0)])
def test_tma_im2col_conv_geometry(N, C, H, M, R, s, p):
    """C % 32 == 0 layers run the TMA im2col engine: strides, paddings, 1x1/3x3/5x5 taps,
    partial pixel tiles and partial N tiles against conv_forward<float>."""
    import torch
    import paper_2003_12203_b200 as F
    from paper_2003_12203_b200 import synth
    D = synth.relu_like((N, C, H, H), 5)
    W = synth.he_normal(M, C, R, 6)
    B = synth.uniform((M,), -0.1, 0.1, 7)
    L = F.ProtectedConv(W, B, F.ConvParams(stride=s, pad=p, bias_enabled=True), N, H)
    Og = L.conv_forward(torch.from_numpy(D).cuda()).cpu().numpy()
    Or = O.conv_f32(O.dims(N, C, H, M, R, s, p, 1, True), D, W, B)
    assert _rel(Og, Or).max() <= 1e-5
    L.close()


@pytest.mark.gpu
def test_act_pool_nhwc_glue_bitwise():
    """ftc_glue_act_pool_nhwc == ftc_glue_act_pool_ck (NCHW output and exact Cd1/Cd2)
    bitwise, and its NHWC output is exactly the channel-last transpose."""
    import torch
    from paper_2003_12203_b200 import _abi
    L = _abi.lib()
    rng = np.random.default_rng(3)
    N, C, H, k, s, p = 3, 64, 27, 3, 2, 0
    Ho = (H + 2 * p - k) // s + 1
    x = torch.from_numpy(rng.standard_normal((N, C, H, H)).astype(np.float32)).cuda()
    out_a = torch.empty((N, C, Ho, Ho), device="cuda")
    out_b = torch.empty_like(out_a)
    nhwc = torch.empty((N, Ho, Ho, C), device="cuda")
    cd = [torch.empty((C, Ho, Ho), dtype=torch.float64, device="cuda") for _ in range(4)]
    st = torch.cuda.current_stream().cuda_stream
    assert L.ftc_glue_act_pool_ck(x.data_ptr(), out_a.data_ptr(), N, C, H, 1, k, s, p, cd[0].data_ptr(),
                                  cd[1].data_ptr(), st) == 0
    assert L.ftc_glue_act_pool_nhwc(x.data_ptr(), out_b.data_ptr(), nhwc.data_ptr(), N, C, H, 1, k, s, p,
                                    cd[2].data_ptr(), cd[3].data_ptr(), st) == 0
    torch.cuda.synchronize()
    assert torch.equal(out_a, out_b)
    assert torch.equal(nhwc, out_b.permute(0, 2, 3, 1))
    assert torch.equal(cd[0], cd[2]) and torch.equal(cd[1], cd[3])


@pytest.mark.gpu
def test_nhwc_staging_guard():
    """A staging declared for one D is ignored when the layer is launched on another D."""
    import torch
    import paper_2003_12203_b200 as F
    from paper_2003_12203_b200 import synth
    N, C, H, M, R = 2, 32, 12, 48, 3
    W = synth.he_normal(M, C, R, 1)
    L = F.ProtectedConv(W, None, F.ConvParams(pad=1), N, H)
    assert L.input_nhwc() is not None
    D1 = torch.from_numpy(synth.relu_like((N, C, H, H), 1)).cuda()
    D2 = torch.from_numpy(synth.relu_like((N, C, H, H), 2)).cuda()
    # declare a staging for D1 (the buffer holds whatever it holds), then run on D2: the
    # launch must restage from D2 rather than trust the declaration
    L.input_nhwc_ready(D1)
    O2 = L.conv_forward(D2).cpu().numpy()
    Or = O.conv_f32(O.dims(N, C, H, M, R, 1, 1, 1, False), D2.cpu().numpy(), W, None)
    assert _rel(O2, Or).max() <= 1e-5
    L.close()


_FUSED_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r}); sys.path.insert(0, {oracle!r})
import paper_2003_12203_b200 as F
from paper_2003_12203_b200 import synth
import oracle_py as O
N, C, H, M, R = 4, 32, 12, 48, 3
D = synth.relu_like((N, C, H, H), 11); W = synth.he_normal(M, C, R, 12); B = synth.uniform((M,), -0.1, 0.1, 13)
L = F.ProtectedConv(W, B, F.ConvParams(pad=1, bias_enabled=True), N, H)
Dg = torch.from_numpy(D).cuda()
plan = F.LayerPlan(rc_enabled=True, clc_enabled=True, tau=1e-3)
O0, rep = L.protected(Dg, plan)
assert not rep.detected
O0 = O0.cpu().numpy()
dims = O.dims(N, C, H, M, R, 1, 1, 1, True)
rng = np.random.default_rng(5)
for t in range(12):
    n, m, x, y = int(rng.integers(N)), int(rng.integers(M)), int(rng.integers(H)), int(rng.integers(H))
    bit = int(rng.integers(20, 31))
    _, r = L.protected(Dg, plan, [F.output_bitflip(n, m, x, y, bit)])
    Os = O0.copy(); Os[n, m, x, y] = synth.flip32(Os[n, m, x, y], bit)
    ref = O.protected_layer(dims, D, W, B, True, True, 1e-3, O_conv=Os)
    got = r.verdict()
    for k in ("detected", "stage", "stages_attempted"):
        assert got[k] == ref[k], (t, k, got, ref)
print("fused ok")
"""


@pytest.mark.gpu
@pytest.mark.parametrize("env_flag", ["", "FTC_NO_FUSED"])
def test_fused_detect_path_verdict_parity(env_flag):
    """Default (fused in-kernel CoC-D) and the side-stream clean path both give the
    reference's verdicts on seeded output flips."""
    env = dict(os.environ)
    if env_flag:
        env[env_flag] = "1"
    code = _FUSED_SCRIPT.format(root=ROOT, oracle=os.path.join(ROOT, "oracle"))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "fused ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.gpu
@pytest.mark.parametrize("N,C,H,act,k,s,p", [(5, 96, 55, 1, 3, 2, 0), (4, 256, 27, 1, 3, 2, 0), (3, 384, 13, 1, 1, 1, 0),
                                             (2, 64, 224, 1, 2, 2, 0), (3, 64, 112, 2, 3, 2, 1), (6, 40, 20, 2, 2, 2, 0),
                                             (17, 32, 56, 0, 1, 1, 0), (2, 3, 227, 0, 1, 1, 0)])
def test_glue_tile_cd1(N, C, H, act, k, s, p):
    """ftc_glue_act_pool_cd1: NCHW output bitwise = ftc_glue_act_pool, NHWC output = its
    channel-last transpose, ws head = sum_n out_n (FP64, any order) -- and identical on a
    second call (the workspace tickets re-arm)."""
    import torch
    from paper_2003_12203_b200 import _abi
    L = _abi.lib()
    rng = np.random.default_rng(N * 1000 + H)
    Ho = (H + 2 * p - k) // s + 1
    x = torch.from_numpy(rng.standard_normal((N, C, H, H)).astype(np.float32)).cuda()
    ref = torch.empty((N, C, Ho, Ho), device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    assert L.ftc_glue_act_pool(x.data_ptr(), ref.data_ptr(), N, C, H, act, k, s, p, None, st) == 0
    nws = L.ftc_glue_ws_doubles(N, C, H, k, s, p)
    assert nws >= C * Ho * Ho
    ws = torch.zeros((nws,), dtype=torch.float64, device="cuda")
    for rep in range(2):
        out = torch.full((N, C, Ho, Ho), float("nan"), device="cuda")
        nhwc = torch.full((N, Ho, Ho, C), float("nan"), device="cuda") if C % 32 == 0 else None
        assert L.ftc_glue_act_pool_cd1(x.data_ptr(), out.data_ptr(), nhwc.data_ptr() if nhwc is not None else None,
                                       N, C, H, act, k, s, p, ws.data_ptr(), st) == 0, _abi.last_error()
        torch.cuda.synchronize()
        assert torch.equal(out, ref)
        if nhwc is not None:
            assert torch.equal(nhwc, ref.permute(0, 2, 3, 1))
        cd1 = ws[:C * Ho * Ho].view(C, Ho, Ho).cpu().numpy()
        exact = ref.double().sum(0).cpu().numpy()
        assert np.abs(cd1 - exact).max() <= 1e-12 * max(1.0, np.abs(exact).max())
        if rep == 0:
            first = cd1.copy()
        else:
            assert np.array_equal(first, cd1)
    # no workspace: outputs only
    out = torch.empty_like(ref)
    assert L.ftc_glue_act_pool_cd1(x.data_ptr(), out.data_ptr(), None, N, C, H, act, k, s, p, None, st) == 0
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


@pytest.mark.gpu
@pytest.mark.parametrize("N,C,H,M,R,s,p,G", [(2, 64, 12, 96, 3, 1, 1, 2), (3, 128, 9, 64, 3, 2, 1, 4),
                                             (2, 96, 11, 48, 1, 1, 0, 3), (2, 12, 10, 24, 3, 1, 1, 3),
                                             (1, 256, 7, 512, 3, 1, 1, 2)])
def test_grouped_conv_on_tensor_cores(N, C, H, M, R, s, p, G):
    """Grouped layers run on the tensor-core engines (TMA im2col when C/groups % 32 == 0,
    register gather otherwise): output vs conv_forward<float>, and a protected call with an
    output flip gives run_protected_layer<double>'s verdict."""
    import torch
    import paper_2003_12203_b200 as F
    from paper_2003_12203_b200 import synth
    D = synth.relu_like((N, C, H, H), 3)
    W = synth.he_normal(M, C // G, R, 4)
    B = synth.uniform((M,), -0.1, 0.1, 5)
    prm = F.ConvParams(stride=s, pad=p, groups=G, bias_enabled=True)
    L = F.ProtectedConv(W, B, prm, N, H)
    Dg = torch.from_numpy(D).cuda()
    Og = L.conv_forward(Dg).cpu().numpy()
    d = O.dims(N, C, H, M, R, s, p, G, True)
    Or = O.conv_f32(d, D, W, B)
    assert _rel(Og, Or).max() <= 1e-5
    plan = F.LayerPlan(rc_enabled=True, clc_enabled=True, tau=1e-3)
    O0, rep = L.protected(Dg, plan)
    assert not rep.detected and torch.equal(O0.cpu(), torch.from_numpy(Og))
    E = Og.shape[-1]
    for t, (n, m, x, y, bit) in enumerate([(0, M - 1, 0, 0, 27), (N - 1, M // G, E - 1, E // 2, 29)]):
        Of, r = L.protected(Dg, plan, [F.output_bitflip(n, m, x, y, bit)])
        Os = Og.copy()
        Os[n, m, x, y] = synth.flip32(Os[n, m, x, y], bit)
        ref = O.protected_layer(d, D, W, B, True, True, 1e-3, O_conv=Os)
        got = r.verdict()
        for k in ("detected", "stage", "stages_attempted"):
            assert got[k] == ref[k], (t, k, got, ref)
        if got["stage"] in ("coc", "rc", "clc", "fc", "recompute"):
            assert np.array_equal(Of.cpu().numpy(), Og)
    L.close()


@pytest.mark.gpu
@pytest.mark.parametrize("N,C,H,M", [(4, 32, 14, 40), (16, 64, 56, 64), (8, 16, 12, 24), (40, 32, 10, 32)])
def test_clean_path_state_across_paths(N, C, H, M):
    """The clean path keeps its device state (Co5 / So5 accumulators, counters) re-armed
    whichever variant a call takes -- Co5 scattered by the staging pass (small batches),
    computed in the conv or after it, or the side-stream path a pre_conv fault selects:
    clean calls interleaved with faulted ones never report a detection."""
    import torch
    import paper_2003_12203_b200 as F
    from paper_2003_12203_b200 import synth
    D = synth.relu_like((N, C, H, H), 21)
    W = synth.he_normal(M, C, 3, 22)
    L = F.ProtectedConv(W, None, F.ConvParams(pad=1), N, H)
    Dg = torch.from_numpy(D).cuda()
    plan = F.LayerPlan(rc_enabled=True, clc_enabled=True, tau=1e-3)
    O0, r = L.protected(Dg, plan)
    assert not r.detected
    seq = [[], [F.Fault("fmap", 1, 2, 3, 4, "add", 0, 5.0)], [], [F.output_bitflip(0, 1, 2, 3, 29)], [],
           [F.Fault("fmap", 0, 0, 0, 0, "add", 0, 7.0)], [], []]
    for k, faults in enumerate(seq):
        O, r = L.protected(Dg, plan, faults)
        if not faults:
            assert not r.detected, (k, r.verdict())
            assert torch.equal(O, O0)
    L.close()
