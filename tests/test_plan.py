"""Per-layer plans and the plan / corpus file formats.

CPU: the library's cost model, RC/ClC decisions, error-probability estimate and default
plan follow test_workflow.cpp:12-44, 236-243, and match the reference live
(oracle/_ref) on random layers; plan JSON and corpus JSONL are byte-identical to the
reference's serialize.cpp output and round-trip (test_model_io.cpp:124-151).
GPU: profile_layer times the six forced-fault workflow variants on the device path
(workflow.hpp:418-501)."""
import math

import numpy as np
import pytest

import oracle_py as O

ref_only = pytest.mark.skipif(not O.have_ref(), reason="needs oracle/_ref (the reference)")


def _P():
    from paper_2003_12203_b200 import plan as P
    return P


def test_cost_model_closed_forms():
    """test_workflow.cpp:12-24"""
    P = _P()
    assert P.cost_model("fc", P.LayerDims()) == 5.0
    d = P.LayerDims(8, 8, 16, 16, 3, 14)
    assert P.cost_model("coc", d) < P.cost_model("fc", d)
    d2 = P.LayerDims(8, 16, 16, 16, 3, 14)
    assert math.isclose(P.cost_model("rc", d2, 1.0, 0.0), 2 * P.cost_model("rc", d, 1.0, 0.0), rel_tol=1e-12)
    # closed forms (workflow.hpp:51-76), every scheme
    N, M, Ch, H, R, E = 3, 5, 7, 11, 3, 9
    d = P.LayerDims(N, M, Ch, H, R, E)
    a, b = 1.5, 0.25
    H2, R2, E2 = H * H, R * R, E * E
    want = {"fc": a * (N + M) * Ch * R2 * E2 + b * (N * Ch * H2 + 2 * N * M * E2),
            "rc": 2 * a * M * Ch * R2 * E2 + 2 * b * (N * Ch * H2 + N * M * E2),
            "clc": 2 * a * N * Ch * R2 * E2 + 2 * b * N * M * E2,
            "coc": 3 * a * Ch * R2 * E2 + b * (2 * N * Ch * H2 + 3 * N * M * E2),
            "coc_d": a * Ch * R2 * E2 + b * (2 * N * Ch * H2 + N * M * E2)}
    for s, v in want.items():
        assert P.cost_model(s, d, a, b) == v, s


def test_rc_decision():
    """test_workflow.cpp:26-37 (equality disables; scale invariant)."""
    P = _P()
    assert P.decide_rc(100, 60, 110, 0.8, 0.2)
    assert not P.decide_rc(100, 100, 110, 0.8, 0.2)
    assert not P.decide_rc(100, 95, 160, 0.5, 0.5)
    assert not P.decide_rc(100, 90, 110, 0.5, 0.5)
    for c in (0.5, 3.0, 1e6):
        assert P.decide_rc(100 * c, 60 * c, 110 * c, 0.8, 0.2)
        assert not P.decide_rc(100 * c, 95 * c, 160 * c, 0.5, 0.5)
    # ClC mirrors it with the probabilities swapped (workflow.hpp:85-88)
    assert P.decide_clc(100, 60, 110, 0.2, 0.8)
    assert not P.decide_clc(100, 60, 110, 0.8, 0.2)


def test_error_probs_follow_element_counts():
    """test_workflow.cpp:39-46"""
    P = _P()
    p_r, p_c = P.estimate_error_probs(P.LayerDims(1, 64, 3, 224, 7, 218))
    assert math.isclose(p_r, 16.0 / 17.0, rel_tol=1e-12)
    assert math.isclose(p_r + p_c, 1.0, rel_tol=1e-15)
    a, _ = P.estimate_error_probs(P.LayerDims(2, 2, 3, 4, 4, 1))
    assert math.isclose(a, 0.5, rel_tol=1e-15)


def test_default_plan_picks_rc_from_cost_model():
    """test_workflow.cpp:236-243"""
    P = _P()
    p = P.make_default_plan(P.LayerDims(8, 4, 3, 32, 3, 30), 1e-4)
    assert p.rc_enabled and not p.clc_enabled and p.tau == 1e-4
    assert not P.make_default_plan(P.LayerDims(2, 32, 3, 16, 3, 14), 1e-4).rc_enabled


def test_default_plan_matches_restatement():
    """The library's default plan == the oracle's restatement, field for field."""
    P = _P()
    rng = np.random.default_rng(7)
    for _ in range(50):
        N, M, Ch, H, R = (int(v) for v in (rng.integers(1, 65), rng.integers(1, 400), rng.integers(1, 400),
                                            rng.integers(3, 230), rng.integers(1, 12)))
        E = max(1, H - R + 1)
        g = P.make_default_plan(P.LayerDims(N, M, Ch, H, R, E), 1e-4)
        w = O.default_plan(N, M, Ch, H, R, E, 1e-4)
        assert (g.rc_enabled, g.clc_enabled) == (w["rc"], w["clc"])
        assert (g.t0, g.t1, g.t2, g.p_r) == (w["t0"], w["t1"], w["t2"], w["p_r"])


@ref_only
def test_default_plan_matches_reference_live():
    import ctypes as C
    P = _P()
    R_ = O.ref()
    rng = np.random.default_rng(8)
    for _ in range(50):
        N, M, Ch, H, R = (int(v) for v in (rng.integers(1, 65), rng.integers(1, 400), rng.integers(1, 400),
                                            rng.integers(3, 230), rng.integers(1, 12)))
        E = max(1, H - R + 1)
        rc, clc = C.c_int(), C.c_int()
        t = [C.c_double() for _ in range(4)]
        R_.ref_make_default_plan(N, M, Ch, H, R, E, C.c_double(1e-4), C.byref(rc), C.byref(clc),
                                 *[C.byref(x) for x in t])
        g = P.make_default_plan(P.LayerDims(N, M, Ch, H, R, E), 1e-4)
        assert (g.rc_enabled, g.clc_enabled) == (bool(rc.value), bool(clc.value))
        assert (g.t0, g.t1, g.t2, g.p_r) == tuple(x.value for x in t)


# ----------------------------------------------------------------------------- file formats
def _plans():
    P = _P()
    return {"c1": P.PlanInfo(True, False, 1e-4, 1.5, 1.0, 2.0, 0.9),
            "conv2": P.make_default_plan(P.LayerDims(128, 256, 96, 27, 5, 27), 1e-4),
            "z": P.PlanInfo(False, True, 1e-10, 0.0, 1e-300, 1e300, 0.1234567890123)}


def test_plan_file_round_trip(tmp_path):
    """test_model_io.cpp:124-142"""
    P = _P()
    from paper_2003_12203_b200.ftconv import IoError
    plans = _plans()
    back = P.plan_from_json(P.plan_to_json(plans))
    assert back == plans
    path = str(tmp_path / "plan.json")
    P.save_plan(path, plans)
    assert P.load_plan(path) == plans
    with pytest.raises(IoError):
        P.plan_from_json("{bad")
    with pytest.raises(IoError):
        P.plan_from_json('{"a": {"rc_enabled": true}}')  # tau is required
    # t0/t1/t2 and p_r are optional (serialize.cpp:135-140)
    p = P.plan_from_json('{"a": {"rc_enabled": true, "clc_enabled": false, "tau": 0.001}}')["a"]
    assert (p.t0, p.t1, p.t2, p.p_r) == (0.0, 0.0, 0.0, 0.5)
    assert p.plan().tau == 1e-3


@ref_only
def test_plan_json_bytes_match_reference():
    P = _P()
    plans = _plans()
    assert P.plan_to_json(plans) == O.ref_plan_to_json({k: v.__dict__ for k, v in plans.items()})


def test_corpus_file_round_trip(tmp_path):
    """test_model_io.cpp:144-151"""
    from paper_2003_12203_b200 import campaign as K
    from paper_2003_12203_b200.ftconv import IoError
    corpus = K.campaign([(2, 4, 3, 8, 3)], 25, seed=11)
    text = K.corpus_to_jsonl(corpus)
    back = K.corpus_from_jsonl(text)
    assert K.corpus_to_jsonl(back) == text
    assert back == corpus
    path = str(tmp_path / "c.jsonl")
    K.save_corpus(path, corpus)
    assert K.load_corpus(path) == corpus
    with pytest.raises(IoError):
        K.corpus_from_jsonl("{not a corpus}\n")
    assert K.corpus_from_jsonl("\n\n") == []


@ref_only
def test_corpus_jsonl_bytes_match_reference():
    from paper_2003_12203_b200 import campaign as K
    for grids, n, seed in [([(2, 4, 3, 8, 3)], 25, 11), ([(4, 6, 3, 9, 3), (1, 1, 2, 5, 1)], 60, 2**63 + 5)]:
        ours = K.corpus_to_jsonl(K.campaign(grids, n, seed=seed))
        theirs = O.ref_corpus_to_jsonl(O.ref_campaign(grids, n, seed=seed))
        assert ours == theirs


# ----------------------------------------------------------------------------- GPU
@pytest.mark.gpu
def test_profile_layer_on_device():
    """workflow.hpp:418-501 on the B200 path: six positive medians; a profiled plan;
    degenerate layers fall back to the cost model; reps < 3 is a ConfigError."""
    import torch
    import paper_2003_12203_b200 as F
    from paper_2003_12203_b200 import synth
    P = _P()
    N, C, H, M, R = 4, 32, 24, 32, 3
    W = synth.he_normal(M, C, R, 4)
    L = F.ProtectedConv(W, None, F.ConvParams(), N, H)
    D = torch.from_numpy(synth.relu_like((N, C, H, H), 3)).cuda()
    pr = P.profile_layer(L, D, 1e-4, reps=5)
    assert not pr.used_cost_model
    ts = (pr.rc_t0, pr.rc_t1, pr.rc_t2, pr.clc_t0, pr.clc_t1, pr.clc_t2)
    assert all(t > 0 for t in ts)
    assert pr.rc_t2 >= pr.rc_t1 * 0.5  # generous noise band (test_workflow.cpp:266-274)
    dims = P.LayerDims.of(L)
    plan = P.plan_from_profile(pr, dims, 1e-4)
    p_r, p_c = P.estimate_error_probs(dims)
    assert plan.rc_enabled == P.decide_rc(pr.rc_t0, pr.rc_t1, pr.rc_t2, p_r, p_c)
    assert plan.clc_enabled == P.decide_clc(pr.clc_t0, pr.clc_t1, pr.clc_t2, p_r, p_c)
    # the layer is left clean: a plain protected run detects nothing afterwards
    _, rep = L.protected(D, plan.plan())
    assert not rep.detected
    with pytest.raises(F.ConfigError):
        P.profile_layer(L, D, 1e-4, reps=2)
    L.close()
    # N = 1: fallback (workflow.hpp:449)
    L1 = F.ProtectedConv(W, None, F.ConvParams(), 1, H)
    pr1 = P.profile_layer(L1, D[:1].contiguous(), 1e-4, reps=3)
    assert pr1.used_cost_model and pr1.rc_t0 > 0
    d1 = P.LayerDims.of(L1)
    assert pr1.rc_t0 == P.cost_model("coc", d1) + P.cost_model("fc", d1)
    L1.close()


def test_tau_policies_from_residuals():
    """nets.taus_from_residuals: all-families = 4x the worst family, power of ten;
    detection = 4x the absolute Co5/So5 residual in the 1-2-5 series, never coarser
    than all-families; floors = tau x median denominator."""
    from paper_2003_12203_b200 import nets
    res = {"a": {"res": [1e-5, 1e-5, 3e-3, 1e-4, 2e-6, 1e-4, 1e-4], "abs5": 4.9e-5, "den5_median": 30.0},
           "b": {"res": [1e-6] * 7, "abs5": 0.5, "den5_median": 2.0}}
    t_all = nets.taus_from_residuals(res, "all-families")
    t_det = nets.taus_from_residuals(res, "detection")
    assert t_all == {"a": 0.1, "b": 1e-5}
    assert t_det["a"] == 2e-4 and t_det["b"] == 1e-5
    fl = nets.detection_floor(res, t_det)
    assert abs(fl["a"] - 2e-4 * 30.0) < 1e-12
    with pytest.raises(ValueError):
        nets.taus_from_residuals(res, "nope")
