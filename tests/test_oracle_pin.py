"""Pin the CPU oracle (oracle/ftc_oracle.c) before trusting it.

1. Known-answer tests restated from the reference's own unit tests
   (proj/tests/test_conv.cpp, test_checksums.cpp, test_schemes.cpp, test_workflow.cpp).
2. Bitwise agreement with the reference itself (oracle/_ref/libftref.so, compiled
   from the unmodified reference headers) on seeded random layers and faults.
These run on CPU (`-m "not gpu"`).
"""
import numpy as np
import pytest

import oracle_py as O

ref_only = pytest.mark.skipif(not O.have_ref(), reason="reference bridge not buildable here")


def rnd(shape, seed, dtype=np.float64):
    return O.tensor_random(shape, seed, dtype=dtype)


# ----------------------------------------------------------------------------- KATs
def test_hand_worked_conv_kat():
    """test_conv.cpp:24-46: 3x3 (*) 2x2 -> [[6,8],[12,14]]; bias 10 -> +10."""
    D = np.arange(1, 10, dtype=np.float64).reshape(1, 1, 3, 3)
    W = np.zeros((1, 1, 2, 2)); W[0, 0, 0, 0] = 1; W[0, 0, 1, 1] = 1
    o = O.conv_f64(O.dims(1, 1, 3, 1, 2), D, W)
    assert o[0, 0].tolist() == [[6, 8], [12, 14]]
    ob = O.conv_f64(O.dims(1, 1, 3, 1, 2, bias=True), D, W, np.array([10.0]))
    assert ob[0, 0].tolist() == [[16, 18], [22, 24]]


def test_identity_and_zero_kernels_kat():
    """test_conv.cpp:48-63."""
    D = rnd((2, 1, 5, 5), 2)
    W = np.ones((1, 1, 1, 1))
    assert np.array_equal(O.conv_f64(O.dims(2, 1, 5, 1, 1), D, W), D)
    D2 = rnd((1, 2, 4, 4), 1)
    assert not O.conv_f64(O.dims(1, 2, 4, 1, 2), D2, np.zeros((1, 2, 2, 2))).any()


def test_extent_rule_kat():
    """test_tensor.cpp:38-50: E=(H+2p-R)/U+1 must be integral."""
    d = O.dims(1, 1, 8, 1, 3, stride=2, pad=0)  # (8-3)%2 != 0
    with pytest.raises(ValueError):
        O.conv_f32(d, np.zeros((1, 1, 8, 8), np.float32), np.zeros((1, 1, 3, 3), np.float32))


def test_kernel_checksum_kat():
    """test_checksums.cpp:59-68: W_m = m*ones -> Cw1 = 3, Cw2 = 5."""
    W = np.zeros((3, 2, 2, 2))
    for m in range(3):
        W[m] = m
    _, _, cw1, cw2 = O.input_checksums(O.dims(1, 2, 2, 3, 2), np.zeros((1, 2, 2, 2)), W)
    assert (cw1 == 3).all() and (cw2 == 5).all()


def test_summation_and_bias_kats():
    """test_checksums.cpp:112-168."""
    Ot = np.zeros((2, 2, 2, 2))
    for n in range(2):
        for m in range(2):
            Ot[n, m] = n + m
    s = O.output_summations(Ot, 16 | 32 | 64)
    assert (s[4] == 4).all() and (s[5] == 3).all() and (s[6] == 3).all()
    s1 = O.output_summations(np.zeros((2, 1, 2, 2)), 1, bias=np.array([3.0]))
    assert (s1[0] == -6).all()
    s3 = O.output_summations(np.zeros((2, 2, 1, 1)), 16 | 32, bias=np.array([1.0, 2.0]))
    assert s3[4][0, 0] == -6 and s3[5][0, 0] == -4


def test_checksum_identities_random_layers():
    """test_checksums.cpp:192-210 (f64, tau=1e-10) incl. groups and bias."""
    rng = np.random.default_rng(777)
    for _ in range(25):
        stride = int(rng.integers(1, 3)); G = int([1, 1, 2, 4][rng.integers(0, 4)])
        R = int([1, 2, 3][rng.integers(0, 3)]); H = R + stride * int(rng.integers(1, 6))
        N = int(rng.integers(1, 5)); Ch = G * int(rng.integers(1, 4)); M = G * int(rng.integers(1, 4))
        bias = bool(rng.integers(0, 2))
        d = O.dims(N, Ch, H, M, R, stride=stride, groups=G, bias=bias)
        D = rnd((N, Ch, H, H), int(rng.integers(1 << 30)))
        W = rnd((M, Ch // G, R, R), int(rng.integers(1 << 30)))
        B = rnd((M,), 5) if bias else None
        cs = O.output_checksums(d, 127, D, W)
        Ou = O.conv_f64(d, D, W, B)
        ss = O.output_summations(Ou, 127, B)
        for c, s_ in zip(cs, ss):
            assert np.all(np.abs(c - s_) <= 1e-10 * np.maximum(1, np.maximum(np.abs(c), np.abs(s_))))


def _wf_fixture(N=3, M=3, seed=500):
    """test_workflow.cpp:51-68 WorkflowFixture (double, tau=1e-10, rc+clc on)."""
    D = rnd((N, 2, 6, 6), seed)
    W = rnd((M, 2, 3, 3), seed + 1)
    d = O.dims(N, 2, 6, M, 3)
    return d, D, W, O.conv_f64(d, D, W)


@pytest.mark.parametrize("case,expect", [
    ("block", ("coc", ["coc"])),
    ("row", ("rc", ["coc", "rc"])),
    ("col", ("clc", ["coc", "rc", "clc"])),
    ("multi", ("recompute", ["coc", "rc", "clc", "fc", "recompute"])),
])
def test_workflow_stage_kats(case, expect):
    """test_workflow.cpp:81-126, 202-216."""
    d, D, W, Oc = _wf_fixture()
    Of = Oc.copy()
    if case == "block":
        Of[1, 2, 0, 0] += 9.0
    elif case == "row":
        for m in range(3):
            Of[1, m, 0, 0] += 2.0 + m
    elif case == "col":
        for n in range(3):
            Of[n, 1, 0, 0] += 2.0 + n
    else:
        Of[0, 1, 0, 0] += 5; Of[0, 2, 0, 0] += 6; Of[1, 1, 1, 1] += 7; Of[2, 1, 0, 1] += 8
    r = O.protected_layer(d, D, W, None, True, True, 1e-10, O_conv=Of, want_output=True)
    assert (r["stage"], r["stages_attempted"]) == expect
    assert np.allclose(r["O"], Oc, atol=1e-8, rtol=0)


def test_workflow_rc_disabled_lands_on_fc():
    d, D, W, Oc = _wf_fixture()
    Of = Oc.copy()
    for m in range(3):
        Of[1, m, 0, 0] += 2.0 + m
    assert O.protected_layer(d, D, W, None, False, False, 1e-10, O_conv=Of)["stage"] == "fc"


@pytest.mark.parametrize("pre,stage,reloaded", [
    ([("W", 1 * 18 + 0, 1, 5.0)], "clc", True),           # kernel fault -> reload + ClC
    ([("cw1", 0 * 9 + 1 * 3 + 1, 1, 4.0)], "reload", True),  # cw1 corruption -> reload
    ([("cd1", 1 * 36 + 2 * 6 + 3, 1, 6.0)], "discard", False),
    ([("cd2", 0, 1, 8.0), ("cw2", 0, 1, 8.0)], "none", False),
    ([("D", 2 * 72 + 0 + 3 * 6 + 3, 1, 4.0)], "rc", False),  # fmap fault row 2 -> RC
    ([("D", 0 * 72 + 0 + 3 * 6 + 3, 1, 4.0)], "discard", False),  # row 0 -> discard
])
def test_workflow_pre_conv_kats(pre, stage, reloaded):
    """test_workflow.cpp:128-200 (pre_conv hooks); the conv runs on the faulted D/W."""
    d, D, W, _ = _wf_fixture()
    r = O.protected_layer(d, D, W, None, True, True, 1e-10, O_conv=None, pre=pre)
    assert r["stage"] == stage
    assert r["weights_reloaded"] == reloaded


def test_no_false_positives_tiny_fp32():
    """test_workflow.cpp:218-234 restated at T=double on FP32 conv outputs."""
    rng = np.random.default_rng(9000)
    for rep in range(300):
        N, M, Ch = (int(rng.integers(1, 4)) for _ in range(3))
        R = int(rng.integers(1, 3)); H = R + 1 + int(rng.integers(0, 4))
        d = O.dims(N, Ch, H, M, R)
        D = O.tensor_random((N, Ch, H, H), rep * 2 + 1, dtype=np.float32)
        W = O.tensor_random((M, Ch, R, R), rep * 2 + 2, dtype=np.float32)
        Of = O.conv_f32(d, D, W)
        assert not O.protected_layer(d, D, W, None, True, False, 1e-4, O_conv=Of)["detected"]


def test_flip_bit_involution():
    """test_fault.cpp:59-91: sign bit excluded (bit % 31), flip twice = identity."""
    for v in (0.5, -1.25, 3.0e-3, 123.0):
        for b in (0, 20, 23, 30, 31, 40):
            f = O.flip_f32(v, b)
            assert O.flip_f32(f, b) == np.float32(v)
            assert np.signbit(f) == np.signbit(np.float32(v))


def test_default_plan_kat():
    """test_workflow.cpp:236-243: N > M layer -> RC on, ClC off."""
    p = O.default_plan(8, 4, 3, 32, 3, 30, 1e-4)
    assert p["rc"] and not p["clc"]


# ----------------------------------------------------------------------------- vs reference
@ref_only
def test_rng_bitwise_vs_reference():
    for seed in (0, 1, 12345, 2**63 + 7):
        assert np.array_equal(O.uniform(seed, 5000), O.uniform(seed, 5000, lib=O.ref()))


@ref_only
def test_conv_and_checksums_bitwise_vs_reference():
    rng = np.random.default_rng(2024)
    tested = 0
    while tested < 40:
        stride = int(rng.integers(1, 3)); R = int([1, 2, 3, 5][rng.integers(0, 4)])
        pad = int(rng.integers(0, 3)); H = int(rng.integers(R, 14))
        if (H + 2 * pad - R) % stride:
            continue
        G = int([1, 1, 2][rng.integers(0, 3)])
        N = int(rng.integers(1, 6)); Ch = G * int(rng.integers(1, 5)); M = G * int(rng.integers(1, 6))
        bias = bool(rng.integers(0, 2))
        d = O.dims(N, Ch, H, M, R, stride, pad, G, bias)
        D = O.tensor_random((N, Ch, H, H), tested * 3 + 1, dtype=np.float32)
        W = O.tensor_random((M, Ch // G, R, R), tested * 3 + 2, dtype=np.float32)
        B = O.tensor_random((M,), tested * 3 + 3, dtype=np.float32) if bias else None
        o1 = O.conv_f32(d, D, W, B)
        assert np.array_equal(o1, O.ref_conv_f32(d, D, W, B)), d
        assert np.array_equal(o1, O.ref_conv_f32(d, D, W, B, impl=1))  # direct == mm (P5)
        Dd, Wd = D.astype(np.float64), W.astype(np.float64)
        for a, b in zip(O.input_checksums(d, Dd, Wd), O.ref_input_checksums(d, Dd, Wd)):
            assert np.array_equal(a, b)
        for a, b in zip(O.output_checksums(d, 127, Dd, Wd), O.ref_output_checksums(d, 127, Dd, Wd)):
            assert np.array_equal(a, b)
        Bd = None if B is None else B.astype(np.float64)
        Od = o1.astype(np.float64)
        for a, b in zip(O.output_summations(Od, 127, Bd), O.ref_output_summations(Od, 127, Bd)):
            assert np.array_equal(a, b)
        tested += 1


def _cmp(a, b):
    keys = ("detected", "stage", "weights_reloaded", "recomputed", "corrected_blocks", "stages_attempted",
            "status")
    return {k: a[k] for k in keys} == {k: b[k] for k in keys}


@ref_only
def test_protected_layer_verdicts_bitwise_vs_reference():
    """run_protected_layer<double> with the O-substituting post_conv hook."""
    rng = np.random.default_rng(31337)
    n_cases = 0
    stages = set()
    for rep in range(120):
        N = int(rng.integers(1, 6)); M = int(rng.integers(1, 6)); Ch = int(rng.integers(1, 5))
        R = int([1, 3][rng.integers(0, 2)]); H = int(rng.integers(R + 1, 10)); pad = int(rng.integers(0, 2))
        bias = bool(rng.integers(0, 2))
        d = O.dims(N, Ch, H, M, R, 1, pad, 1, bias)
        E = O.extent(d)
        D = O.tensor_random((N, Ch, H, H), rep * 5 + 1, dtype=np.float32)
        W = O.tensor_random((M, Ch, R, R), rep * 5 + 2, dtype=np.float32)
        B = O.tensor_random((M,), rep * 5 + 3, dtype=np.float32) if bias else None
        Oc = O.conv_f32(d, D, W, B)
        Of = Oc.copy()
        kind = rep % 4
        nflip = 1 if kind == 0 else int(rng.integers(1, 4))
        for _ in range(nflip):
            n = int(rng.integers(0, N)) if kind != 2 else 0
            m = int(rng.integers(0, M)) if kind != 3 else 0
            if kind == 2:
                n = int(rng.integers(0, N))
            x, y = int(rng.integers(0, E)), int(rng.integers(0, E))
            Of[n, m, x, y] = O.flip_f32(Of[n, m, x, y], int(rng.integers(20, 31)))
        rc, clc = bool(rng.integers(0, 2)), bool(rng.integers(0, 2))
        tau = float([1e-3, 1e-4, 1e-5][rng.integers(0, 3)])
        a = O.protected_layer(d, D, W, B, rc, clc, tau, O_conv=Of, want_output=True)
        b = O.ref_protected_layer(d, D, W, B, rc, clc, tau, O_conv=Of, want_output=True)
        assert _cmp(a, b), (rep, a, b)
        if a["status"] == 0:
            assert np.array_equal(a["O"], b["O"], equal_nan=True)
        stages.add(a["stage"])
        n_cases += 1
    assert {"coc", "recompute"} <= stages


@ref_only
def test_pre_conv_faults_bitwise_vs_reference():
    rng = np.random.default_rng(99)
    for rep in range(40):
        N, M, Ch = 3, 3, 2
        d = O.dims(N, Ch, 6, M, 3)
        D = O.tensor_random((N, Ch, 6, 6), rep + 11, dtype=np.float32)
        W = O.tensor_random((M, Ch, 3, 3), rep + 12, dtype=np.float32)
        tgt = ["D", "W", "cd1", "cd2", "cw1", "cw2"][rep % 6]
        size = {"D": D.size, "W": W.size, "cd1": Ch * 36, "cd2": Ch * 36, "cw1": Ch * 9, "cw2": Ch * 9}[tgt]
        pre = [(tgt, int(rng.integers(0, size)), 1, float(rng.uniform(0.5, 5.0)))]
        a = O.protected_layer(d, D, W, None, True, bool(rep % 2), 1e-9, O_conv=None, pre=pre)
        b = O.ref_protected_layer(d, D, W, None, True, bool(rep % 2), 1e-9, O_conv=None, pre=pre)
        assert _cmp(a, b), (rep, tgt, a, b)
