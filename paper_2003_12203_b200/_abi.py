"""ctypes binding of include/ftc_abi.h (libftconv_b200.so).

The library is REQUIRED: importing the compute entry points without it raises.
There is no CPU path; every call lands in hand-written sm_100a kernels.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FTC_LIB_PATH") or os.path.join(PKG, "libftconv_b200.so")  # override: experiments only

MAX_BLOCKS = 4096
MAX_STAGES = 8

# every symbol include/ftc_abi.h declares (checked by tests/test_abi_symbols.py)
EXPORTS = (
    "ftc_abi_version", "ftc_last_error", "ftc_set_conv_engine", "ftc_get_conv_engine",
    "ftc_output_extent", "ftc_layer_create", "ftc_layer_destroy", "ftc_layer_extent",
    "ftc_conv_forward", "ftc_protected_conv", "ftc_protected_conv_host",
    "ftc_protected_conv_launch", "ftc_protected_conv_finish", "ftc_input_checksums",
    "ftc_kernel_checksums", "ftc_output_checksums", "ftc_output_summations", "ftc_detect_coc_d",
    "ftc_verify_kernel", "ftc_layer_set_timing", "ftc_layer_kernel_time", "ftc_kernel_launches",
    "ftc_glue_act_pool", "ftc_glue_add_act", "ftc_glue_pad_crop", "ftc_protected_conv_launch_ck",
    "ftc_glue_act_pool_ck", "ftc_conv_forward_host", "ftc_protected_check",
    "ftc_layer_input_nhwc", "ftc_layer_input_nhwc_ready", "ftc_glue_act_pool_nhwc",
    "ftc_campaign", "ftc_ground_truth_of", "ftc_spec_faults", "ftc_conv_forward_faulted",
    "ftc_cost_model", "ftc_decide_rc", "ftc_decide_clc", "ftc_estimate_error_probs", "ftc_make_default_plan",
    "ftc_profile_layer", "ftc_layer_desc", "ftc_glue_ws_doubles", "ftc_glue_act_pool_cd1",
    "ftc_protected_conv_launch_cd1", "ftc_mt64_uniform", "ftc_conv_backward", "ftc_protected_backward",
    "ftc_conv_backward_host", "ftc_protected_backward_host", "ftc_isolated_scheme",
    "ftc_protected_conv_cancel", "ftc_layer_detect_record", "ftc_protected_conv_peek",
    "ftc_glue_nchw_optional",
    "ftc_device_alloc", "ftc_device_free", "ftc_memcpy", "ftc_memset_zero",
)


class ConvDesc(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("N", "C", "H", "M", "R", "stride", "pad", "groups",
                                         "bias_enabled")]


class GradFault(C.Structure):
    _fields_ = [("target", C.c_int32), ("mode", C.c_int32), ("index", C.c_int64), ("value", C.c_double)]


class BackwardReport(C.Structure):
    _fields_ = [("dw_detected", C.c_int32), ("dd_detected", C.c_int32), ("recomputed", C.c_int32)]


class Plan(C.Structure):
    _fields_ = [("rc_enabled", C.c_int32), ("clc_enabled", C.c_int32), ("tau", C.c_double),
                ("t0", C.c_double), ("t1", C.c_double), ("t2", C.c_double), ("p_r", C.c_double)]


class Fault(C.Structure):
    _fields_ = [("target", C.c_int32), ("mode", C.c_int32), ("n", C.c_int32), ("m", C.c_int32),
                ("x", C.c_int32), ("y", C.c_int32), ("bit", C.c_uint32), ("value", C.c_float),
                ("n_coef", C.c_float), ("m_coef", C.c_float), ("seed", C.c_uint64)]


class FaultSpec(C.Structure):
    _fields_ = [("layer_index", C.c_int32), ("target", C.c_int32), ("checksum", C.c_int32), ("mode", C.c_int32),
                ("i", C.c_int64), ("j", C.c_int64), ("x", C.c_int64), ("y", C.c_int64), ("bit", C.c_uint32),
                ("pad_", C.c_uint32), ("seed", C.c_uint64)]


class GroundTruth(C.Structure):
    _fields_ = [("benign", C.c_int32), ("expected_stage", C.c_int32), ("output_diverges", C.c_int32)]


class LayerGrid(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("N", "M", "Ch", "H", "R")]


class LayerDims(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("N", "M", "Ch", "H", "R", "E")]


class PlanInfo(C.Structure):
    _fields_ = [("rc_enabled", C.c_int32), ("clc_enabled", C.c_int32), ("tau", C.c_double), ("t0", C.c_double),
                ("t1", C.c_double), ("t2", C.c_double), ("p_r", C.c_double)]


class ProfileResult(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("rc_t0", "rc_t1", "rc_t2", "clc_t0", "clc_t1", "clc_t2")] + \
        [("used_cost_model", C.c_int32)]


class Report(C.Structure):
    _fields_ = [("detected", C.c_int32), ("stage", C.c_int32), ("weights_reloaded", C.c_int32),
                ("recomputed", C.c_int32), ("n_blocks", C.c_int32),
                ("blocks", (C.c_int32 * 2) * MAX_BLOCKS), ("n_stages", C.c_int32),
                ("stages", C.c_int32 * MAX_STAGES), ("max_rel_dev", C.c_double),
                ("n_flagged", C.c_int32), ("repaired_planes", C.c_int32),
                ("t_detect_ms", C.c_double), ("t_total_ms", C.c_double)]


_lib = None


def lib():
    """Load the CUDA library; fail loudly if it was not built (no fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: run `python paper_2003_12203_b200/build.py` "
                "(or __graft_entry__.build()); this package has no CPU fallback")
        L = C.CDLL(LIB_PATH)
        vp, i32, u32, dbl = C.c_void_p, C.c_int32, C.c_uint32, C.c_double
        L.ftc_last_error.restype = C.c_char_p
        L.ftc_abi_version.restype = i32
        L.ftc_layer_create.argtypes = [C.POINTER(ConvDesc), vp, vp, C.POINTER(vp)]
        L.ftc_layer_destroy.argtypes = [vp]
        L.ftc_layer_extent.argtypes = [vp, C.POINTER(i32)]
        L.ftc_output_extent.argtypes = [i32, i32, i32, i32, C.POINTER(i32)]
        L.ftc_conv_forward.argtypes = [vp, vp, vp, vp]
        L.ftc_protected_conv.argtypes = [vp, C.POINTER(Plan), vp, vp, C.POINTER(Fault), i32,
                                         C.POINTER(Report), vp]
        L.ftc_protected_conv_host.argtypes = L.ftc_protected_conv.argtypes
        L.ftc_protected_check.argtypes = [vp, C.POINTER(Plan), vp, vp, C.POINTER(Report), vp]
        L.ftc_protected_conv_launch.argtypes = [vp, C.POINTER(Plan), vp, vp, C.POINTER(Fault), i32,
                                                vp]
        L.ftc_protected_conv_finish.argtypes = [vp, C.POINTER(Report)]
        L.ftc_protected_conv_cancel.argtypes = [vp]
        L.ftc_layer_detect_record.argtypes = [vp, vp, vp]
        L.ftc_isolated_scheme.argtypes = [vp, C.POINTER(Plan), vp, vp, C.POINTER(Fault), i32, i32,
                                          C.POINTER(i32), C.POINTER(Report), vp]
        L.ftc_input_checksums.argtypes = [C.POINTER(ConvDesc), vp, vp, vp, vp]
        L.ftc_kernel_checksums.argtypes = [C.POINTER(ConvDesc), vp, vp, vp, vp]
        L.ftc_output_checksums.argtypes = [C.POINTER(ConvDesc), u32, vp, vp, vp, vp, vp, vp,
                                           C.POINTER(vp), vp]
        L.ftc_output_summations.argtypes = [i32, i32, i32, vp, u32, vp, C.POINTER(vp), vp]
        L.ftc_detect_coc_d.argtypes = [vp, vp, i32, dbl, vp, C.POINTER(i32), C.POINTER(dbl), vp]
        L.ftc_verify_kernel.argtypes = [C.POINTER(ConvDesc), vp, vp, dbl, C.POINTER(i32), vp]
        L.ftc_set_conv_engine.argtypes = [C.c_int]
        L.ftc_layer_set_timing.argtypes = [vp, i32]
        L.ftc_layer_kernel_time.argtypes = [vp, C.POINTER(dbl), C.POINTER(i32), i32]
        L.ftc_kernel_launches.restype = C.c_uint64
        L.ftc_glue_act_pool.argtypes = [vp, vp, i32, i32, i32, i32, i32, i32, i32, C.POINTER(i32), vp]
        L.ftc_protected_conv_launch_ck.argtypes = [vp, C.POINTER(Plan), vp, vp, vp, vp, C.POINTER(Fault),
                                                   i32, vp]
        L.ftc_glue_act_pool_ck.argtypes = [vp, vp, i32, i32, i32, i32, i32, i32, i32, vp, vp, vp]
        L.ftc_glue_act_pool_nhwc.argtypes = [vp, vp, vp, i32, i32, i32, i32, i32, i32, i32, vp, vp, vp]
        L.ftc_layer_input_nhwc.argtypes = [vp, C.POINTER(vp)]
        L.ftc_layer_input_nhwc_ready.argtypes = [vp, vp]
        L.ftc_campaign.argtypes = [C.POINTER(LayerGrid), i32, C.c_int64, C.POINTER(dbl), C.c_uint64,
                                   C.POINTER(FaultSpec), C.POINTER(GroundTruth)]
        L.ftc_ground_truth_of.argtypes = [C.POINTER(FaultSpec), C.c_int64, C.c_int64, C.POINTER(GroundTruth)]
        L.ftc_spec_faults.argtypes = [C.POINTER(FaultSpec), C.POINTER(Fault), C.POINTER(i32)]
        L.ftc_conv_forward_faulted.argtypes = [vp, vp, vp, C.POINTER(Fault), i32, vp]
        L.ftc_cost_model.argtypes = [i32, C.POINTER(LayerDims), dbl, dbl]
        L.ftc_cost_model.restype = dbl
        L.ftc_decide_rc.argtypes = [dbl] * 5
        L.ftc_decide_clc.argtypes = [dbl] * 5
        L.ftc_estimate_error_probs.argtypes = [C.POINTER(LayerDims), C.POINTER(dbl), C.POINTER(dbl)]
        L.ftc_estimate_error_probs.restype = None
        L.ftc_make_default_plan.argtypes = [C.POINTER(LayerDims), dbl, dbl, dbl, C.POINTER(PlanInfo)]
        L.ftc_profile_layer.argtypes = [vp, vp, dbl, i32, C.POINTER(ProfileResult), vp]
        L.ftc_layer_desc.argtypes = [vp, vp]
        L.ftc_glue_add_act.argtypes = [vp, vp, vp, C.c_int64, i32, vp]
        L.ftc_mt64_uniform.argtypes = [C.c_uint64, dbl, dbl, C.c_int64, vp]
        L.ftc_conv_backward.argtypes = [C.POINTER(ConvDesc), vp, vp, vp, vp, vp, vp]
        L.ftc_protected_backward.argtypes = [C.POINTER(ConvDesc), vp, vp, vp, dbl, C.POINTER(GradFault), i32, vp,
                                             vp, C.POINTER(BackwardReport), vp]
        L.ftc_glue_ws_doubles.argtypes = [i32] * 6
        L.ftc_glue_ws_doubles.restype = C.c_int64
        L.ftc_glue_act_pool_cd1.argtypes = [vp, vp, vp, i32, i32, i32, i32, i32, i32, i32, vp, vp]
        L.ftc_glue_nchw_optional.argtypes = [vp, i32, i32, i32, i32, i32]
        L.ftc_glue_nchw_optional.restype = i32
        L.ftc_protected_conv_peek.argtypes = [vp, C.POINTER(i32)]
        L.ftc_protected_conv_launch_cd1.argtypes = [vp, C.POINTER(Plan), vp, vp, vp, C.POINTER(Fault), i32, vp]
        L.ftc_glue_pad_crop.argtypes = [vp, vp, i32, i32, i32, i32, i32, vp]
        L.ftc_device_alloc.argtypes = [C.c_size_t, C.POINTER(vp)]
        L.ftc_device_free.argtypes = [vp]
        L.ftc_memcpy.argtypes = [vp, vp, C.c_size_t, i32, vp]
        L.ftc_memset_zero.argtypes = [vp, C.c_size_t, vp]
        _lib = L
    return _lib


def last_error() -> str:
    return lib().ftc_last_error().decode(errors="replace")
