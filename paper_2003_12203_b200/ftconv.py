"""Reference-shaped Python API over the C ABI (names mirror proj/core/include/ftconv/).

    ConvParams, LayerPlan, LayerReport, ResolveStage      (tensor.hpp, workflow.hpp, report.hpp)
    ShapeError, ConfigError, IoError, IntegrityError      (errors.hpp)
    output_extent, conv_forward, run_protected_layer      (tensor.hpp, conv.hpp, workflow.hpp)
    input_checksums, kernel_checksums, output_checksums,
    output_summations, detect_coc_d, verify_kernel        (checksums.hpp, schemes.hpp)
    FaultSpec helpers -> ftc_fault lists                  (fault.hpp)
    ProtectedConv: a layer handle (the per-layer state build_model precomputes)

Device tensors are torch CUDA tensors (torch is plumbing for memory and streams);
numpy arrays are accepted by the *_host entry points.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _abi

STAGES = ["none", "reload", "coc", "rc", "clc", "fc", "discard", "recompute"]


class FtcError(RuntimeError):
    pass


class ShapeError(FtcError):
    pass


class ConfigError(FtcError):
    pass


class IoError(FtcError):
    pass


class IntegrityError(FtcError):
    pass


class CudaError(FtcError):
    pass


_ERRS = {1: ShapeError, 2: ConfigError, 3: IoError, 4: IntegrityError, 5: CudaError, 6: ValueError}


def _check(status: int, what: str):
    if status:
        raise _ERRS.get(status, FtcError)(f"{what}: {_abi.last_error()}")


@dataclass
class ConvParams:
    """tensor.hpp:92-97"""
    stride: int = 1
    groups: int = 1
    pad: int = 0
    bias_enabled: bool = False


@dataclass
class LayerPlan:
    """workflow.hpp:23-29"""
    rc_enabled: bool = True
    clc_enabled: bool = False
    tau: float = 1e-4
    t0: float = 0.0
    t1: float = 0.0
    t2: float = 0.0
    p_r: float = 0.5

    def c(self) -> _abi.Plan:
        return _abi.Plan(int(self.rc_enabled), int(self.clc_enabled), self.tau, self.t0, self.t1,
                         self.t2, self.p_r)


@dataclass
class LayerReport:
    """report.hpp:38-47 (+ device-side diagnostics)"""
    layer: str = ""
    detected: bool = False
    stage: str = "none"
    weights_reloaded: bool = False
    recomputed: bool = False
    corrected_blocks: list = field(default_factory=list)
    stages_attempted: list = field(default_factory=list)
    max_rel_dev: float = 0.0
    n_flagged: int = 0
    n_blocks: int = 0
    repaired_planes: int = 0
    timings: dict = field(default_factory=dict)
    integrity_error: bool = False  # recompute failed twice (the reference throws IntegrityError)

    @staticmethod
    def from_c(r: _abi.Report) -> "LayerReport":
        nb = min(r.n_blocks, _abi.MAX_BLOCKS)
        return LayerReport(
            detected=bool(r.detected), stage=STAGES[r.stage], weights_reloaded=bool(r.weights_reloaded),
            recomputed=bool(r.recomputed),
            corrected_blocks=[(r.blocks[b][0], r.blocks[b][1]) for b in range(nb)],
            stages_attempted=[STAGES[r.stages[s]] for s in range(r.n_stages)],
            max_rel_dev=r.max_rel_dev, n_flagged=r.n_flagged, n_blocks=r.n_blocks,
            repaired_planes=r.repaired_planes,
            timings={"detect_ms": r.t_detect_ms, "total_ms": r.t_total_ms})

    def verdict(self) -> dict:
        return {"detected": self.detected, "stage": self.stage,
                "weights_reloaded": self.weights_reloaded, "recomputed": self.recomputed,
                "corrected_blocks": list(self.corrected_blocks),
                "stages_attempted": list(self.stages_attempted)}


# ----------------------------------------------------------------------------- faults (fault.hpp)
TARGETS = {"output": 0, "fmap": 1, "kernel": 2, "cd1": 3, "cd2": 4, "cw1": 5, "cw2": 6}
MODES = {"bitflip": 0, "add": 1, "set": 2, "scale": 3}


@dataclass
class Fault:
    """One injected fault (FaultSpec, fault.hpp:42-53, as a substitution the device applies)."""
    target: str = "output"
    n: int = -1
    m: int = -1
    x: int = -1
    y: int = -1
    mode: str = "bitflip"
    bit: int = 23
    value: float = 0.0
    n_coef: float = 0.0
    m_coef: float = 0.0
    seed: int = 0  # scale mode: the FaultSpec seed (mt19937_64 magnitudes, fault.hpp:72-80)

    def c(self) -> _abi.Fault:
        return _abi.Fault(TARGETS[self.target], MODES[self.mode], self.n, self.m, self.x, self.y,
                          self.bit, self.value, self.n_coef, self.m_coef, self.seed & (2**64 - 1))


def output_bitflip(n, m, x, y, bit) -> Fault:
    return Fault("output", n, m, x, y, "bitflip", bit)


def _faults_c(faults):
    faults = list(faults or [])
    arr = (_abi.Fault * max(1, len(faults)))()
    for i, f in enumerate(faults):
        arr[i] = f.c() if isinstance(f, Fault) else f
    return arr, len(faults)


# ----------------------------------------------------------------------------- helpers
def _torch():
    import torch
    return torch


def _ptr(t) -> int:
    return 0 if t is None else t.data_ptr()


def _check_tensor(t, shape, what: str, dtype=None):
    """Device tensors cross the C ABI as raw pointers: check device, dtype, layout and
    shape first (a CPU, fp16, strided or undersized tensor would otherwise be read or
    written out of bounds on the device).  Raises ShapeError like the reference's
    check_conv_shapes (conv.hpp:16-37)."""
    torch = _torch()
    dtype = dtype or torch.float32
    if not isinstance(t, torch.Tensor):
        raise ShapeError(f"{what}: expected a torch CUDA tensor, got {type(t).__name__}")
    if not t.is_cuda:
        raise ShapeError(f"{what}: tensor must live on a CUDA device")
    if t.dtype != dtype:
        raise ShapeError(f"{what}: dtype {t.dtype}, expected {dtype}")
    if not t.is_contiguous():
        raise ShapeError(f"{what}: tensor must be contiguous")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ShapeError(f"{what}: shape {tuple(t.shape)}, expected {tuple(shape)}")


def _stream_ptr(stream) -> int:
    if stream is None:
        return _torch().cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def output_extent(H: int, R: int, p: ConvParams) -> int:
    """tensor.hpp:100-107"""
    E = C.c_int32()
    _check(_abi.lib().ftc_output_extent(H, R, p.pad, p.stride, C.byref(E)), "output_extent")
    return E.value


def desc(N, Cin, H, M, R, p: ConvParams) -> _abi.ConvDesc:
    return _abi.ConvDesc(N, Cin, H, M, R, p.stride, p.pad, p.groups, int(p.bias_enabled))


def set_conv_engine(name: str) -> None:
    """'tc' (tcgen05 3xTF32, default) or 'simt' (FP32 FFMA)."""
    _check(_abi.lib().ftc_set_conv_engine({"tc": 0, "simt": 1}[name]), "set_conv_engine")


# ----------------------------------------------------------------------------- layer handle
class ProtectedConv:
    """One protected conv layer bound to a batch size: golden W/bias on device, golden
    Cw1/Cw2 precomputed (model.hpp:104), packed tensor-core operands, scratch."""

    def __init__(self, W: np.ndarray, bias: np.ndarray | None, p: ConvParams, N: int, H: int):
        W = np.ascontiguousarray(W, np.float32)
        if W.ndim != 4 or W.shape[2] != W.shape[3]:
            raise ShapeError("kernel must be M x Ckw x R x R")
        self.M, Ckw, self.R, _ = W.shape
        self.C = Ckw * p.groups
        self.N, self.H, self.p = N, H, p
        if p.bias_enabled:
            if bias is None or np.asarray(bias).size != self.M:
                raise ShapeError("bias length must equal kernel count M")
            bias = np.ascontiguousarray(np.asarray(bias).reshape(-1), np.float32)
        else:
            bias = None
        self._W = W
        self._bias = bias
        self.desc = desc(N, self.C, H, self.M, self.R, p)
        h = C.c_void_p()
        _check(_abi.lib().ftc_layer_create(C.byref(self.desc), W.ctypes.data,
                                           bias.ctypes.data if bias is not None else None,
                                           C.byref(h)), "ftc_layer_create")
        self.h = h
        E = C.c_int32()
        _abi.lib().ftc_layer_extent(self.h, C.byref(E))
        self.E = E.value

    def close(self):
        if getattr(self, "h", None):
            _abi.lib().ftc_layer_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def out_shape(self):
        return (self.N, self.M, self.E, self.E)

    @property
    def in_shape(self):
        return (self.N, self.C, self.H, self.H)

    def _io(self, D, O):
        _check_tensor(D, self.in_shape, "D")
        _check_tensor(O, self.out_shape, "O")
        if O.device != D.device:
            raise ShapeError("D and O must live on the same device")

    def _cd(self, cd, what):
        _check_tensor(cd, (self.C, self.H, self.H), what, _torch().float64)

    def _empty_out(self, D):
        torch = _torch()
        return torch.empty(self.out_shape, dtype=torch.float32, device=D.device)

    def input_nhwc(self):
        """Device pointer of the layer's NHWC input staging buffer (TMA im2col engine) or None."""
        p = C.c_void_p()
        _check(_abi.lib().ftc_layer_input_nhwc(self.h, C.byref(p)), "input_nhwc")
        return p.value

    def input_nhwc_ready(self, D):
        """Declare that the staging buffer already holds D (NHWC) for the next launch on D."""
        _check(_abi.lib().ftc_layer_input_nhwc_ready(self.h, _ptr(D)), "input_nhwc_ready")

    def conv_forward(self, D, O=None, stream=None):
        """conv_forward(D, W, bias, p) on device (conv.hpp:114-131)."""
        O = self._empty_out(D) if O is None else O
        self._io(D, O)
        _check(_abi.lib().ftc_conv_forward(self.h, _ptr(D), _ptr(O), _stream_ptr(stream)),
               "ftc_conv_forward")
        return O

    def protected(self, D, plan: LayerPlan, faults=(), O=None, stream=None):
        """run_protected_layer (workflow.hpp:141-339) on device tensors -> (O, LayerReport)."""
        O = self._empty_out(D) if O is None else O
        self._io(D, O)
        arr, n = _faults_c(faults)
        rep = _abi.Report()
        pl = plan.c()
        st = _abi.lib().ftc_protected_conv(self.h, C.byref(pl), _ptr(D), _ptr(O), arr, n,
                                           C.byref(rep), _stream_ptr(stream))
        if st == 4:  # FTC_INTEGRITY_ERROR
            # the reference throws after filling the report (workflow.hpp:325-338); keep it
            err = IntegrityError(f"ftc_protected_conv: {_abi.last_error()}")
            err.report = LayerReport.from_c(rep)
            raise err
        _check(st, "ftc_protected_conv")
        return O, LayerReport.from_c(rep)

    def check(self, D, O, plan: LayerPlan, stream=None) -> LayerReport:
        """run_protected_layer on an output O produced elsewhere (post_conv substitution);
        O is repaired in place."""
        self._io(D, O)
        rep = _abi.Report()
        pl = plan.c()
        _check(_abi.lib().ftc_protected_check(self.h, C.byref(pl), _ptr(D), _ptr(O), C.byref(rep),
                                              _stream_ptr(stream)), "ftc_protected_check")
        return LayerReport.from_c(rep)

    def isolated(self, D, plan: LayerPlan, scheme: str, faults=(), O=None, stream=None):
        """One scheme in isolation (acceptance.cpp:207-292): detection + reload preamble,
        then only `scheme` ("coc" | "rc" | "clc" | "fc") with a Co5-only verifier.
        Returns (O, status, LayerReport); status is "clean" (settled by the preamble),
        "corrected", "discard" or "escalate"."""
        O = self._empty_out(D) if O is None else O
        self._io(D, O)
        arr, n = _faults_c(faults)
        rep = _abi.Report()
        pl = plan.c()
        st = C.c_int32()
        code = {"coc": 1, "rc": 2, "clc": 3, "fc": 4}[scheme]
        _check(_abi.lib().ftc_isolated_scheme(self.h, C.byref(pl), _ptr(D), _ptr(O), arr, n, code, C.byref(st),
                                              C.byref(rep), _stream_ptr(stream)), "ftc_isolated_scheme")
        names = {-1: "clean", 0: "corrected", 1: "discard", 2: "escalate"}
        return O, names[st.value], LayerReport.from_c(rep)

    def launch(self, D, O, plan: LayerPlan, faults=(), stream=None):
        self._io(D, O)
        arr, n = _faults_c(faults)
        self._pl = plan.c()
        _check(_abi.lib().ftc_protected_conv_launch(self.h, C.byref(self._pl), _ptr(D), _ptr(O), arr,
                                                    n, _stream_ptr(stream)), "launch")

    def launch_ck(self, D, O, cd1, cd2, plan: LayerPlan, faults=(), stream=None):
        """launch with exact input checksums supplied by D's producer (FP64 device tensors)."""
        self._io(D, O)
        self._cd(cd1, "cd1")
        self._cd(cd2, "cd2")
        arr, n = _faults_c(faults)
        self._pl = plan.c()
        _check(_abi.lib().ftc_protected_conv_launch_ck(self.h, C.byref(self._pl), _ptr(D), _ptr(O), _ptr(cd1),
                                                       _ptr(cd2), arr, n, _stream_ptr(stream)), "launch_ck")

    def launch_cd1(self, D, O, cd1, plan: LayerPlan, faults=(), stream=None):
        """launch with the clean-path checksum Cd1 = sum_n D_n (FP64, any order) supplied by
        D's producer, e.g. the start of an ftc_glue_act_pool_cd1 workspace."""
        self._io(D, O)
        _check_tensor(cd1, None, "cd1", _torch().float64)
        if cd1.numel() < self.C * self.H * self.H:
            raise ShapeError("cd1: workspace smaller than C*H*H")
        arr, n = _faults_c(faults)
        self._pl = plan.c()
        _check(_abi.lib().ftc_protected_conv_launch_cd1(self.h, C.byref(self._pl), _ptr(D), _ptr(O), _ptr(cd1),
                                                        arr, n, _stream_ptr(stream)), "launch_cd1")

    def peek_flagged(self) -> int:
        """Wait for the in-flight call's clean path; > 0 when finish() will run the error
        path (ftc_protected_conv_peek).  The call stays in flight."""
        n = C.c_int32(0)
        _check(_abi.lib().ftc_protected_conv_peek(self.h, C.byref(n)), "peek")
        return int(n.value)

    def cancel(self) -> None:
        """Drop the call in flight without judging it (its input was stale)."""
        _check(_abi.lib().ftc_protected_conv_cancel(self.h), "cancel")

    def finish(self) -> LayerReport:
        rep = _abi.Report()
        st = _abi.lib().ftc_protected_conv_finish(self.h, C.byref(rep))
        if st == 4:  # FTC_INTEGRITY_ERROR: the report is filled (workflow.hpp:325-338)
            err = IntegrityError(f"finish: {_abi.last_error()}")
            err.report = LayerReport.from_c(rep)
            raise err
        _check(st, "finish")
        return LayerReport.from_c(rep)

    def protected_host(self, D: np.ndarray, plan: LayerPlan, faults=(), O: np.ndarray | None = None,
                       stream=None):
        """Host buffers in/out (the reference's calling convention)."""
        D = np.ascontiguousarray(D, np.float32)
        O = np.empty(self.out_shape, np.float32) if O is None else O
        arr, n = _faults_c(faults)
        rep = _abi.Report()
        pl = plan.c()
        st = _abi.lib().ftc_protected_conv_host(self.h, C.byref(pl), D.ctypes.data, O.ctypes.data,
                                                arr, n, C.byref(rep),
                                                0 if stream is None else _stream_ptr(stream))
        _check(st, "ftc_protected_conv_host")
        return O, LayerReport.from_c(rep)


# ----------------------------------------------------------------------------- one-shot API
def _to_dev(a):
    torch = _torch()
    if isinstance(a, np.ndarray):
        return torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()
    return a.contiguous()


def conv_forward(D, W, bias, p: ConvParams):
    """conv.hpp:114-131 (device tensors or numpy in, torch CUDA tensor out)."""
    Dd = _to_dev(D)
    Wn = W.cpu().numpy() if hasattr(W, "cpu") else np.asarray(W)
    bn = None if bias is None else (bias.cpu().numpy() if hasattr(bias, "cpu") else np.asarray(bias))
    layer = ProtectedConv(Wn, bn, p, Dd.shape[0], Dd.shape[2])
    try:
        return layer.conv_forward(Dd)
    finally:
        torch = _torch()
        torch.cuda.synchronize()
        layer.close()


@dataclass
class BackwardReport:
    """workflow.hpp:343-347"""
    dw_detected: bool = False
    dd_detected: bool = False
    recomputed: bool = False


@dataclass
class GradFault:
    """The reference's post_hook (workflow.hpp:350-353) as a substitution on the first
    pass: dW or dD element `index` (flat NCHW) set to / incremented by `value`."""
    target: str = "dW"  # "dW" | "dD"
    index: int = 0
    mode: str = "add"   # "set" | "add"
    value: float = 0.0

    def c(self) -> _abi.GradFault:
        return _abi.GradFault(0 if self.target == "dW" else 1, 0 if self.mode == "set" else 1, int(self.index),
                              float(self.value))


def _bwd_setup(D, W, dO, p: ConvParams):
    torch = _torch()
    Dd, Wd, gd = _to_dev(D), _to_dev(W), _to_dev(dO)
    N, Cin, H = Dd.shape[0], Dd.shape[1], Dd.shape[2]
    M, R = Wd.shape[0], Wd.shape[2]
    d = desc(N, Cin, H, M, R, ConvParams(stride=p.stride, pad=p.pad, groups=p.groups, bias_enabled=False))
    if p.groups != 1:
        raise ConfigError("grouped back-propagation is unsupported")
    E = output_extent(H, R, p)
    if tuple(gd.shape) != (N, M, E, E) or Wd.shape[1] != Cin or Wd.shape[3] != R or Dd.shape[3] != H:
        raise ShapeError("upstream gradient shape must be N x M x E x E")
    dW = torch.empty((M, Cin, R, R), dtype=torch.float32, device=Dd.device)
    dD = torch.empty((N, Cin, H, H), dtype=torch.float32, device=Dd.device)
    return d, Dd, Wd, gd, dW, dD


def conv_backward(D, W, dO, p: ConvParams, stream=None):
    """conv_backward (conv.hpp:150-185) -> (dW, dD) on the device (FP64 accumulation)."""
    d, Dd, Wd, gd, dW, dD = _bwd_setup(D, W, dO, p)
    _check(_abi.lib().ftc_conv_backward(C.byref(d), _ptr(Dd), _ptr(Wd), _ptr(gd), _ptr(dW), _ptr(dD),
                                        _stream_ptr(stream)), "conv_backward")
    return dW, dD


def run_protected_backward(D, W, dO, p: ConvParams, tau: float, faults=(), stream=None):
    """run_protected_backward (workflow.hpp:350-417) -> (dW, dD, BackwardReport);
    IntegrityError (with .report) when the recompute fails verification."""
    d, Dd, Wd, gd, dW, dD = _bwd_setup(D, W, dO, p)
    faults = list(faults or ())
    arr = (_abi.GradFault * max(1, len(faults)))(*[f.c() for f in faults])
    rep = _abi.BackwardReport()
    st = _abi.lib().ftc_protected_backward(C.byref(d), _ptr(Dd), _ptr(Wd), _ptr(gd), float(tau), arr, len(faults),
                                           _ptr(dW), _ptr(dD), C.byref(rep), _stream_ptr(stream))
    out = BackwardReport(bool(rep.dw_detected), bool(rep.dd_detected), bool(rep.recomputed))
    if st == 4:  # FTC_INTEGRITY_ERROR
        err = IntegrityError(f"run_protected_backward: {_abi.last_error()}")
        err.report = out
        raise err
    _check(st, "run_protected_backward")
    return dW, dD, out


def run_protected_layer(D, W, bias, p: ConvParams, plan: LayerPlan, faults=()):
    """workflow.hpp:141-339 -> (O, LayerReport)."""
    Dd = _to_dev(D)
    Wn = W.cpu().numpy() if hasattr(W, "cpu") else np.asarray(W)
    bn = None if bias is None else (bias.cpu().numpy() if hasattr(bias, "cpu") else np.asarray(bias))
    layer = ProtectedConv(Wn, bn, p, Dd.shape[0], Dd.shape[2])
    try:
        return layer.protected(Dd, plan, faults)
    finally:
        layer.close()


def input_checksums(D, W, groups: int, stream=None):
    """checksums.hpp:91-113 -> (cd1, cd2, cw1, cw2) FP64 device tensors."""
    torch = _torch()
    N, Cin, H, _ = D.shape
    M, Ckw, R, _ = W.shape
    d = _abi.ConvDesc(N, Cin, H, M, R, 1, 0, groups, 0)
    cd1 = torch.empty((Cin, H, H), dtype=torch.float64, device=D.device)
    cd2 = torch.empty_like(cd1)
    cw1 = torch.empty((Cin, R, R), dtype=torch.float64, device=D.device)
    cw2 = torch.empty_like(cw1)
    s = _stream_ptr(stream)
    _check(_abi.lib().ftc_input_checksums(C.byref(d), _ptr(D), _ptr(cd1), _ptr(cd2), s), "input_checksums")
    _check(_abi.lib().ftc_kernel_checksums(C.byref(d), _ptr(W), _ptr(cw1), _ptr(cw2), s), "kernel_checksums")
    return cd1, cd2, cw1, cw2


def output_checksums(which: int, D, W, ic, p: ConvParams, stream=None):
    """checksums.hpp:134-161 -> list of 7 FP64 device tensors (None where not requested)."""
    torch = _torch()
    N, Cin, H, _ = D.shape
    M, Ckw, R, _ = W.shape
    E = output_extent(H, R, p)
    d = desc(N, Cin, H, M, R, p)
    shapes = [(M, E, E), (N, E, E), (M, E, E), (N, E, E), (E, E), (E, E), (E, E)]
    out = [torch.empty(s, dtype=torch.float64, device=D.device) if which & (1 << k) else None
           for k, s in enumerate(shapes)]
    arr = (C.c_void_p * 7)(*[_ptr(o) or None for o in out])
    cd1, cd2, cw1, cw2 = ic
    _check(_abi.lib().ftc_output_checksums(C.byref(d), which, _ptr(D), _ptr(W), _ptr(cd1), _ptr(cd2),
                                           _ptr(cw1), _ptr(cw2), arr, _stream_ptr(stream)),
           "output_checksums")
    return out


def output_summations(O, which: int, bias=None, stream=None):
    """checksums.hpp:165-245 -> list of 7 FP64 device tensors (bias-adjusted if bias given)."""
    torch = _torch()
    N, M, E, _ = O.shape
    shapes = [(M, E, E), (N, E, E), (M, E, E), (N, E, E), (E, E), (E, E), (E, E)]
    out = [torch.empty(s, dtype=torch.float64, device=O.device) if which & (1 << k) else None
           for k, s in enumerate(shapes)]
    arr = (C.c_void_p * 7)(*[_ptr(o) or None for o in out])
    _check(_abi.lib().ftc_output_summations(N, M, E, _ptr(O), which, _ptr(bias), arr, _stream_ptr(stream)),
           "output_summations")
    return out


def detect_coc_d(co5, so5, tau: float, stream=None):
    """schemes.hpp:79-94 -> (clean, mismatch_mask (uint8 device), max_rel_dev)."""
    torch = _torch()
    mask = torch.empty(co5.numel(), dtype=torch.uint8, device=co5.device)
    clean = C.c_int32()
    mrd = C.c_double()
    _check(_abi.lib().ftc_detect_coc_d(_ptr(co5), _ptr(so5), co5.numel(), tau, _ptr(mask), C.byref(clean),
                                       C.byref(mrd), _stream_ptr(stream)), "detect_coc_d")
    return bool(clean.value), mask, mrd.value


def verify_kernel(W, cw1_ref, groups: int, tau: float, C_in: int | None = None, stream=None) -> bool:
    """checksums.hpp:250-259"""
    M, Ckw, R, _ = W.shape
    d = _abi.ConvDesc(1, Ckw * groups, R, M, R, 1, 0, groups, 0)
    ok = C.c_int32()
    _check(_abi.lib().ftc_verify_kernel(C.byref(d), _ptr(W), _ptr(cw1_ref), tau, C.byref(ok),
                                        _stream_ptr(stream)), "verify_kernel")
    return bool(ok.value)
