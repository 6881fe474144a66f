"""Checksum-protected back-propagation (conv.hpp:150-185,
workflow.hpp:340-417).

CPU: the oracle's restatement is pinned bitwise against the reference itself and
against the reference's own backward test cases (test_conv.cpp:149-228,
test_workflow.cpp:276-309).  GPU: gradients against the oracle (FP64) and torch,
verdicts (dw_detected / dd_detected / recomputed) identical to the oracle's
run_protected_backward<double> on the same FP32 inputs and the same hook."""
import numpy as np
import pytest

import oracle_py as O

ref_only = pytest.mark.skipif(not O.have_ref(), reason="needs oracle/_ref (the reference)")


def _random_case(rng):
    while True:
        N, M, C, R = (int(v) for v in rng.integers(1, 4, 4))
        H = int(rng.integers(R, 9))
        s, p = int(rng.integers(1, 3)), int(rng.integers(0, 2))
        if (H + 2 * p - R) % s == 0:
            return O.dims(N, C, H, M, R, s, p)


@ref_only
def test_oracle_backward_pinned_to_reference():
    rng = np.random.default_rng(11)
    for t in range(40):
        d = _random_case(rng)
        E = O.extent(d)
        D = rng.standard_normal((d.N, d.C, d.H, d.H))
        W = rng.standard_normal((d.M, d.C, d.R, d.R))
        dO = rng.standard_normal((d.N, d.M, E, E))
        a, b = O.conv_backward(d, D, W, dO), O.conv_backward(d, D, W, dO, lib=O.ref())
        assert a[0] == b[0] == 0 and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
        hooks = ([("dW", int(rng.integers(d.M * d.C * d.R * d.R)), "add", 2.5)] if t % 3 == 0 else
                 [("dD", int(rng.integers(d.N * d.C * d.H * d.H)), "set", 7.0)] if t % 3 == 1 else [])
        x = O.protected_backward(d, D, W, dO, 1e-10, hooks)
        y = O.protected_backward(d, D, W, dO, 1e-10, hooks, lib=O.ref())
        assert x[0] == y[0] and x[3] == y[3]
        assert np.array_equal(x[1], y[1]) and np.array_equal(x[2], y[2])


def test_oracle_backward_reference_kats():
    # test_conv.cpp:149-158 scalar case
    d = O.dims(1, 1, 1, 1, 1)
    st, dW, dD = O.conv_backward(d, np.array([[[[3.0]]]]), np.array([[[[5.0]]]]), np.array([[[[7.0]]]]))
    assert st == 0 and dW.item() == 21 and dD.item() == 35
    # :160-175 ones upstream gradient sums input windows
    D = np.arange(1, 10, dtype=np.float64).reshape(1, 1, 3, 3)
    W = O.tensor_random((1, 1, 2, 2), 11, dtype=np.float64)
    st, dW, _ = O.conv_backward(O.dims(1, 1, 3, 1, 2), D, W, np.ones((1, 1, 2, 2)))
    for i in range(2):
        for j in range(2):
            assert abs(dW[0, 0, i, j] - D[0, 0, i:i + 2, j:j + 2].sum()) <= 1e-12
    # :177-186 zero upstream gradient
    d = O.dims(2, 2, 4, 3, 2)
    st, dW, dD = O.conv_backward(d, O.tensor_random((2, 2, 4, 4), 12, dtype=np.float64),
                                 O.tensor_random((3, 2, 2, 2), 13, dtype=np.float64), np.zeros((2, 3, 3, 3)))
    assert not dW.any() and not dD.any()
    # :220-228 grouped params -> ConfigError
    st, _, _ = O.conv_backward(O.dims(1, 2, 4, 2, 2, 1, 0, 2), np.zeros((1, 2, 4, 4)), np.zeros((2, 1, 2, 2)),
                               np.zeros((1, 2, 3, 3)))
    assert st == 2
    # test_workflow.cpp:276-309
    d = O.dims(2, 2, 5, 3, 2)
    D = O.tensor_random((2, 2, 5, 5), 10, dtype=np.float64)
    W = O.tensor_random((3, 2, 2, 2), 11, dtype=np.float64)
    dO = O.tensor_random((2, 3, 4, 4), 12, dtype=np.float64)
    st, dW, dD, f = O.protected_backward(d, D, W, dO, 1e-10)
    _, rw, rd = O.conv_backward(d, D, W, dO)
    assert st == 0 and not any(f.values()) and np.array_equal(dW, rw) and np.array_equal(dD, rd)
    idx_w = ((1 * 2 + 0) * 2 + 0) * 2 + 0
    st, dW, _, f = O.protected_backward(d, D, W, dO, 1e-10, [("dW", idx_w, "add", 3.0)])
    assert f["dw_detected"] and f["recomputed"] and np.array_equal(dW, rw)
    idx_d = ((0 * 2 + 1) * 5 + 2) * 5 + 2
    st, _, dD, f = O.protected_backward(d, D, W, dO, 1e-10, [("dD", idx_d, "add", -4.0)])
    assert f["dd_detected"] and f["recomputed"] and np.array_equal(dD, rd)


def _close(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return (np.abs(a - b) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))).max(initial=0.0)


@pytest.mark.gpu
def test_gpu_conv_backward_vs_oracle():
    import torch
    import paper_2003_12203_b200 as F
    rng = np.random.default_rng(21)
    for _ in range(25):
        d = _random_case(rng)
        E = O.extent(d)
        D = rng.standard_normal((d.N, d.C, d.H, d.H)).astype(np.float32)
        W = rng.standard_normal((d.M, d.C, d.R, d.R)).astype(np.float32)
        dO = rng.standard_normal((d.N, d.M, E, E)).astype(np.float32)
        dW, dD = F.conv_backward(D, W, dO, F.ConvParams(stride=d.stride, pad=d.pad))
        torch.cuda.synchronize()
        _, rw, rd = O.conv_backward(d, D, W, dO)
        assert _close(dW.cpu().numpy(), rw) <= 1e-6 and _close(dD.cpu().numpy(), rd) <= 1e-6


@pytest.mark.gpu
@pytest.mark.parametrize("N,C,H,M,R,s,p", [(16, 64, 56, 64, 3, 1, 1), (4, 3, 227, 96, 11, 4, 0), (8, 96, 27, 64, 5, 1, 2)])
def test_gpu_conv_backward_large_vs_torch(N, C, H, M, R, s, p):
    """BASELINE-shaped layers against torch's FP64 conv2d gradients"""
    import torch
    import paper_2003_12203_b200 as F
    g = torch.Generator(device="cuda").manual_seed(N + H)
    D = torch.randn((N, C, H, H), device="cuda", generator=g)
    W = torch.randn((M, C, R, R), device="cuda", generator=g) * (2.0 / (C * R * R)) ** 0.5
    E = (H + 2 * p - R) // s + 1
    dO = torch.randn((N, M, E, E), device="cuda", generator=g)
    dW, dD = F.conv_backward(D, W, dO, F.ConvParams(stride=s, pad=p))
    D64, W64, g64 = D.double(), W.double(), dO.double()
    rw = torch.nn.grad.conv2d_weight(D64, W64.shape, g64, stride=s, padding=p)
    rd = torch.nn.grad.conv2d_input(D64.shape, W64, g64, stride=s, padding=p)
    torch.cuda.synchronize()
    assert _close(dW.cpu().numpy(), rw.cpu().numpy()) <= 1e-6
    assert _close(dD.cpu().numpy(), rd.cpu().numpy()) <= 1e-6


@pytest.mark.gpu
def test_gpu_protected_backward_verdict_parity():
    import torch
    import paper_2003_12203_b200 as F
    rng = np.random.default_rng(707)
    for t in range(30):
        d = _random_case(rng)
        E = O.extent(d)
        D = rng.standard_normal((d.N, d.C, d.H, d.H)).astype(np.float32)
        W = rng.standard_normal((d.M, d.C, d.R, d.R)).astype(np.float32)
        dO = rng.standard_normal((d.N, d.M, E, E)).astype(np.float32)
        kind = t % 4
        hooks = []
        if kind == 1:
            hooks = [("dW", int(rng.integers(d.M * d.C * d.R * d.R)), "add", 2.5)]
        elif kind == 2:
            hooks = [("dD", int(rng.integers(d.N * d.C * d.H * d.H)), "add", -4.0)]
        elif kind == 3:
            hooks = [("dW", int(rng.integers(d.M * d.C * d.R * d.R)), "set", 1e3),
                     ("dD", int(rng.integers(d.N * d.C * d.H * d.H)), "add", 1e-3)]
        faults = [F.GradFault(tg, i, m, v) for tg, i, m, v in hooks]
        dW, dD, rep = F.run_protected_backward(D, W, dO, F.ConvParams(stride=d.stride, pad=d.pad), 1e-10, faults)
        torch.cuda.synchronize()
        st, rw, rd, flags = O.protected_backward(d, D, W, dO, 1e-10, hooks)
        assert st == 0
        assert {"dw_detected": rep.dw_detected, "dd_detected": rep.dd_detected,
                "recomputed": rep.recomputed} == flags, (t, hooks)
        # outputs are the clean gradients either way (repaired by the recompute)
        _, cw, cd = O.conv_backward(d, D, W, dO)
        assert _close(dW.cpu().numpy(), cw) <= 1e-6 and _close(dD.cpu().numpy(), cd) <= 1e-6


@pytest.mark.gpu
def test_gpu_backward_errors():
    import torch
    import paper_2003_12203_b200 as F
    D = torch.zeros((1, 2, 4, 4), device="cuda")
    with pytest.raises(F.ShapeError):
        F.conv_backward(D, torch.zeros((2, 2, 2, 2), device="cuda"), torch.zeros((1, 2, 2, 2), device="cuda"),
                        F.ConvParams())
    with pytest.raises(F.ConfigError):
        F.conv_backward(D, torch.zeros((2, 1, 2, 2), device="cuda"), torch.zeros((1, 2, 3, 3), device="cuda"),
                        F.ConvParams(groups=2))
