"""Per-layer protection plans.

Mirrors the reference's plan interface (workflow.hpp:19-112, 418-501; serialize.cpp:
115-155): ``cost_model``, ``decide_rc`` / ``decide_clc``, ``estimate_error_probs``,
``make_default_plan`` (host arithmetic in the library), ``profile_layer`` (the six
forced-fault variants timed on the device path) and the plan file format.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass

from . import _abi
from .ftconv import LayerPlan, ProtectedConv, _check, _ptr, _stream_ptr

SCHEMES = ("coc_d", "coc", "rc", "clc", "fc")


@dataclass
class LayerDims:
    """workflow.hpp:38-40"""
    N: int = 1
    M: int = 1
    Ch: int = 1
    H: int = 1
    R: int = 1
    E: int = 1

    def c(self) -> _abi.LayerDims:
        return _abi.LayerDims(self.N, self.M, self.Ch, self.H, self.R, self.E)

    @staticmethod
    def of(layer: ProtectedConv) -> "LayerDims":
        d = layer.desc
        return LayerDims(d.N, d.M, d.C, d.H, d.R, layer.out_shape[-1])


@dataclass
class PlanInfo:
    """LayerPlan with its profiled runtimes (workflow.hpp:22-28)."""
    rc_enabled: bool = True
    clc_enabled: bool = False
    tau: float = 1e-4
    t0: float = 0.0
    t1: float = 0.0
    t2: float = 0.0
    p_r: float = 0.5

    def plan(self) -> LayerPlan:
        return LayerPlan(rc_enabled=self.rc_enabled, clc_enabled=self.clc_enabled, tau=self.tau)


@dataclass
class ProfileResult:
    """workflow.hpp:423-427"""
    rc_t0: float = 0.0
    rc_t1: float = 0.0
    rc_t2: float = 0.0
    clc_t0: float = 0.0
    clc_t1: float = 0.0
    clc_t2: float = 0.0
    used_cost_model: bool = False


def cost_model(scheme: str, dims: LayerDims, alpha: float = 1.0, beta: float = 1.0) -> float:
    return _abi.lib().ftc_cost_model(SCHEMES.index(scheme), C.byref(dims.c()), alpha, beta)


def decide_rc(t0, t1, t2, p_r, p_c) -> bool:
    return bool(_abi.lib().ftc_decide_rc(t0, t1, t2, p_r, p_c))


def decide_clc(t0, t1, t2, p_r, p_c) -> bool:
    return bool(_abi.lib().ftc_decide_clc(t0, t1, t2, p_r, p_c))


def estimate_error_probs(dims: LayerDims):
    pr, pc = C.c_double(), C.c_double()
    _abi.lib().ftc_estimate_error_probs(C.byref(dims.c()), C.byref(pr), C.byref(pc))
    return pr.value, pc.value


def make_default_plan(dims: LayerDims, tau: float, alpha: float = 1.0, beta: float = 1.0) -> PlanInfo:
    o = _abi.PlanInfo()
    _check(_abi.lib().ftc_make_default_plan(C.byref(dims.c()), tau, alpha, beta, C.byref(o)), "make_default_plan")
    return PlanInfo(bool(o.rc_enabled), bool(o.clc_enabled), o.tau, o.t0, o.t1, o.t2, o.p_r)


def profile_layer(layer: ProtectedConv, D, tau: float, reps: int = 5, stream=None) -> ProfileResult:
    o = _abi.ProfileResult()
    _check(_abi.lib().ftc_profile_layer(layer.h, _ptr(D), tau, reps, C.byref(o), _stream_ptr(stream)),
           "profile_layer")
    return ProfileResult(o.rc_t0, o.rc_t1, o.rc_t2, o.clc_t0, o.clc_t1, o.clc_t2, bool(o.used_cost_model))


def plan_from_profile(pr: ProfileResult, dims: LayerDims, tau: float) -> PlanInfo:
    """Profiled plan: RC and ClC decided on the measured workflow times."""
    p_r, p_c = estimate_error_probs(dims)
    rc = decide_rc(pr.rc_t0, pr.rc_t1, pr.rc_t2, p_r, p_c)
    clc = decide_clc(pr.clc_t0, pr.clc_t1, pr.clc_t2, p_r, p_c)
    return PlanInfo(rc, clc, tau, pr.rc_t0, pr.rc_t1, pr.rc_t2, p_r)


# ----------------------------------------------------------------------------- plan files
def plan_to_json(plans: dict) -> str:
    """serialize.cpp:115-124 (keys sorted, 2-space indent, trailing newline)."""
    obj = {name: {"clc_enabled": p.clc_enabled, "p_r": p.p_r, "rc_enabled": p.rc_enabled, "t0": p.t0,
                  "t1": p.t1, "t2": p.t2, "tau": p.tau} for name, p in plans.items()}
    return json.dumps(obj, indent=2, sort_keys=True) + "\n"


def plan_from_json(text: str) -> dict:
    """serialize.cpp:126-146 (t0/t1/t2 default 0, p_r 0.5)."""
    try:
        j = json.loads(text)
        return {name: PlanInfo(bool(v["rc_enabled"]), bool(v["clc_enabled"]), float(v["tau"]),
                               float(v.get("t0", 0.0)), float(v.get("t1", 0.0)), float(v.get("t2", 0.0)),
                               float(v.get("p_r", 0.5))) for name, v in j.items()}
    except (ValueError, KeyError, TypeError, AttributeError) as e:
        from .ftconv import IoError
        raise IoError(f"malformed plan file: {e}")


def save_plan(path: str, plans: dict) -> None:
    with open(path, "w") as f:
        f.write(plan_to_json(plans))


def load_plan(path: str) -> dict:
    with open(path) as f:
        return plan_from_json(f.read())
