"""ctypes view of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Loads oracle/libftc_oracle.so (the C restatement of the reference path) and, when
present, oracle/_ref/libftref.so (the reference itself, compiled from its headers
by oracle/Makefile).  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs import this module; the product package
never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libftc_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libftref.so")
MAX_BLOCKS = 4096

STAGES = ["none", "reload", "coc", "rc", "clc", "fc", "discard", "recompute"]
CK = {f"O{k}": 1 << (k - 1) for k in range(1, 8)}
CK_ALL = 127

_lock = threading.Lock()


class Dims(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("N", "C", "H", "M", "R", "stride", "pad", "groups", "bias")]


class Report(C.Structure):
    _fields_ = [
        ("detected", C.c_int), ("stage", C.c_int), ("weights_reloaded", C.c_int),
        ("recomputed", C.c_int), ("n_blocks", C.c_int), ("blocks", (C.c_int * 2) * MAX_BLOCKS),
        ("n_stages", C.c_int), ("stages", C.c_int * 8), ("max_rel_dev", C.c_double),
    ]

    def as_dict(self) -> dict:
        nb = min(self.n_blocks, MAX_BLOCKS)
        return {
            "detected": bool(self.detected),
            "stage": STAGES[self.stage],
            "weights_reloaded": bool(self.weights_reloaded),
            "recomputed": bool(self.recomputed),
            "corrected_blocks": [(self.blocks[b][0], self.blocks[b][1]) for b in range(nb)],
            "n_blocks": int(self.n_blocks),
            "stages_attempted": [STAGES[self.stages[s]] for s in range(self.n_stages)],
        }


class PreFault(C.Structure):
    _fields_ = [("target", C.c_int), ("index", C.c_longlong), ("mode", C.c_int), ("value", C.c_double)]


PRE_TARGETS = {"D": 0, "W": 1, "cd1": 2, "cd2": 3, "cw1": 4, "cw2": 5}


def build() -> None:
    """Compile the oracle (and the reference bridge when /root/reference exists)."""
    with _lock:
        subprocess.run(["make", "-s", "-C", HERE], check=True)


def _load(path: str):
    return C.CDLL(path)


_OR = None
_REF = None


def oracle():
    global _OR
    if _OR is None:
        if not os.path.exists(ORACLE_SO):
            build()
        _OR = _load(ORACLE_SO)
    return _OR


def have_ref() -> bool:
    if not os.path.exists(REF_SO) and os.path.isdir("/root/reference/proj/core/include"):
        build()
    return os.path.exists(REF_SO)


def ref():
    global _REF
    if _REF is None:
        if not have_ref():
            raise RuntimeError("oracle/_ref/libftref.so not available")
        _REF = _load(REF_SO)
    return _REF


def P(a: np.ndarray | None, ctype=C.c_double):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ctype))


def dims(N, Cin, H, M, R, stride=1, pad=0, groups=1, bias=False) -> Dims:
    return Dims(N, Cin, H, M, R, stride, pad, groups, int(bool(bias)))


def extent(d: Dims) -> int:
    return (d.H + 2 * d.pad - d.R) // d.stride + 1


# ----------------------------------------------------------------------------- generators
def uniform(seed: int, n: int, lo=-1.0, hi=1.0, lib=None) -> np.ndarray:
    out = np.empty(n, np.float64)
    L = lib or oracle()
    fn = L.or_mt64_uniform if L is oracle() else L.ref_mt64_uniform
    fn.argtypes = [C.c_uint64, C.c_double, C.c_double, C.c_size_t, C.POINTER(C.c_double)]
    fn(C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), lo, hi, n, P(out))
    return out


def tensor_random(shape, seed, lo=-1.0, hi=1.0, dtype=np.float32) -> np.ndarray:
    """Tensor4<T>::random (tensor.hpp:57-66): draws in double, casts to T."""
    n = int(np.prod(shape))
    return uniform(seed, n, lo, hi).astype(dtype).reshape(shape)


# ----------------------------------------------------------------------------- oracle calls
def conv_f32(d: Dims, D: np.ndarray, W: np.ndarray, bias=None) -> np.ndarray:
    L = oracle()
    E = extent(d)
    O = np.empty((d.N, d.M, E, E), np.float32)
    b = None if bias is None else np.ascontiguousarray(bias, np.float32)
    st = L.or_conv_forward_f32(C.byref(d), P(np.ascontiguousarray(D, np.float32), C.c_float),
                               P(np.ascontiguousarray(W, np.float32), C.c_float),
                               P(b, C.c_float), P(O, C.c_float))
    if st:
        raise ValueError(f"or_conv_forward_f32 status {st}")
    return O


def conv_f64(d: Dims, D, W, bias=None) -> np.ndarray:
    L = oracle()
    E = extent(d)
    O = np.empty((d.N, d.M, E, E), np.float64)
    b = None if bias is None else np.ascontiguousarray(bias, np.float64)
    st = L.or_conv_forward_f64(C.byref(d), P(np.ascontiguousarray(D, np.float64)),
                               P(np.ascontiguousarray(W, np.float64)), P(b), P(O))
    if st:
        raise ValueError(f"or_conv_forward_f64 status {st}")
    return O


def input_checksums(d: Dims, D, W):
    L = oracle()
    D = np.ascontiguousarray(D, np.float64)
    W = np.ascontiguousarray(W, np.float64)
    cd1 = np.empty((d.C, d.H, d.H)); cd2 = np.empty_like(cd1)
    cw1 = np.empty((d.C, d.R, d.R)); cw2 = np.empty_like(cw1)
    L.or_input_checksums(C.byref(d), P(D), P(cd1), P(cd2))
    L.or_kernel_checksums(C.byref(d), P(W), P(cw1), P(cw2))
    return cd1, cd2, cw1, cw2


def _fam_shapes(N, M, E):
    return [(M, E, E), (N, E, E), (M, E, E), (N, E, E), (E, E), (E, E), (E, E)]


def output_checksums(d: Dims, which: int, D, W):
    L = oracle()
    D = np.ascontiguousarray(D, np.float64)
    W = np.ascontiguousarray(W, np.float64)
    cd1, cd2, cw1, cw2 = input_checksums(d, D, W)
    E = extent(d)
    out = [np.zeros(s) if which & (1 << k) else None for k, s in enumerate(_fam_shapes(d.N, d.M, E))]
    arr = (C.POINTER(C.c_double) * 7)(*[P(o) if o is not None else None for o in out])
    st = L.or_output_checksums(C.byref(d), C.c_uint(which), P(D), P(W), P(cd1), P(cd2), P(cw1), P(cw2), arr)
    if st:
        raise ValueError(f"or_output_checksums status {st}")
    return out


def output_summations(O: np.ndarray, which: int, bias=None):
    L = oracle()
    N, M, E, _ = O.shape
    O = np.ascontiguousarray(O, np.float64)
    out = [np.zeros(s) if which & (1 << k) else None for k, s in enumerate(_fam_shapes(N, M, E))]
    arr = (C.POINTER(C.c_double) * 7)(*[P(o) if o is not None else None for o in out])
    b = None if bias is None else np.ascontiguousarray(bias, np.float64)
    L.or_output_summations(N, M, E, P(O), C.c_uint(which), P(b), arr)
    return out


def _f64(a):
    """FP32 arrays are widened exactly; float64 arrays pass through."""
    if a is None:
        return None
    a = np.asarray(a)
    if a.dtype == np.float64:
        return np.ascontiguousarray(a)
    return np.ascontiguousarray(a, np.float32).astype(np.float64)


def _pre_array(pre):
    pre = pre or []
    arr = (PreFault * max(1, len(pre)))()
    for i, (t, idx, mode, val) in enumerate(pre):
        arr[i] = PreFault(PRE_TARGETS[t] if isinstance(t, str) else t, idx, mode, val)
    return arr, len(pre)


def protected_layer(d: Dims, D, W, bias, rc: bool, clc: bool, tau: float, O_conv=None, pre=None,
                    want_output=False, O_recompute=None):
    """run_protected_layer<double> restated; O_conv = the post_conv hook's output.

    Inputs D/W/bias are FP32 arrays widened exactly to double."""
    L = oracle()
    Dd, Wd, bd, Od = _f64(D), _f64(W), _f64(bias), _f64(O_conv)

    class Plan(C.Structure):
        _fields_ = [("rc_enabled", C.c_int), ("clc_enabled", C.c_int), ("tau", C.c_double)]

    pl = Plan(int(rc), int(clc), tau)
    pre_arr, npre = _pre_array(pre)
    rep = Report()
    E = extent(d)
    Oout = np.empty((d.N, d.M, E, E)) if want_output else None
    Orc = _f64(O_recompute)
    st = L.or_protected_layer_seam(C.byref(d), P(Dd), P(Wd), P(bd), C.byref(pl), P(Od), P(Orc), pre_arr,
                                   npre, C.byref(rep), P(Oout))
    res = rep.as_dict()
    res["status"] = st
    res["max_rel_dev"] = rep.max_rel_dev
    if want_output:
        res["O"] = Oout
    return res


def isolated_scheme(d: Dims, D, W, bias, tau, O_conv, scheme: str, want_output=False):
    L = oracle()
    code = {"coc": 1, "rc": 2, "clc": 3, "fc": 4}[scheme]
    Dd, Wd, bd, Od = _f64(D), _f64(W), _f64(bias), _f64(O_conv)
    nb = C.c_int(0)
    blocks = np.zeros(2 * MAX_BLOCKS, np.int32)
    E = extent(d)
    Oout = np.empty((d.N, d.M, E, E)) if want_output else None
    L.or_isolated_scheme.restype = C.c_int
    st = L.or_isolated_scheme(C.byref(d), P(Dd), P(Wd), P(bd), C.c_double(tau), P(Od), code, P(Oout),
                              C.byref(nb), P(blocks, C.c_int))
    names = {-1: "clean", 0: "corrected", 1: "discard", 2: "escalate"}
    res = {"status": names.get(st, st), "blocks": [(int(blocks[2 * b]), int(blocks[2 * b + 1]))
                                                   for b in range(min(nb.value, MAX_BLOCKS))]}
    if want_output:
        res["O"] = Oout
    return res


def flip_f32(v: float, bit: int) -> np.float32:
    u = np.array([v], np.float32).view(np.uint32)
    u ^= np.uint32(1 << (bit % 31))
    return u.view(np.float32)[0]


def default_plan(N, M, Ch, H, R, E, tau):
    L = oracle()
    rc = C.c_int(); clc = C.c_int(); t0 = C.c_double(); t1 = C.c_double(); t2 = C.c_double(); pr = C.c_double()
    L.or_make_default_plan(N, M, Ch, H, R, E, C.c_double(tau), C.byref(rc), C.byref(clc), C.byref(t0),
                           C.byref(t1), C.byref(t2), C.byref(pr))
    return {"rc": bool(rc.value), "clc": bool(clc.value), "t0": t0.value, "t1": t1.value,
            "t2": t2.value, "p_r": pr.value}


# ----------------------------------------------------------------------------- reference calls
def ref_conv_f32(d: Dims, D, W, bias=None, impl=0) -> np.ndarray:
    R_ = ref()
    E = extent(d)
    O = np.empty((d.N, d.M, E, E), np.float32)
    b = None if bias is None else np.ascontiguousarray(bias, np.float32)
    st = R_.ref_conv_forward_f32(C.byref(d), P(np.ascontiguousarray(D, np.float32), C.c_float),
                                 P(np.ascontiguousarray(W, np.float32), C.c_float), P(b, C.c_float),
                                 P(O, C.c_float), impl)
    if st:
        raise ValueError(f"ref_conv_forward_f32 status {st}")
    return O


def ref_output_checksums(d: Dims, which: int, D, W):
    R_ = ref()
    E = extent(d)
    out = [np.zeros(s) if which & (1 << k) else None for k, s in enumerate(_fam_shapes(d.N, d.M, E))]
    arr = (C.POINTER(C.c_double) * 7)(*[P(o) if o is not None else None for o in out])
    st = R_.ref_output_checksums(C.byref(d), C.c_uint(which), P(np.ascontiguousarray(D, np.float64)),
                                 P(np.ascontiguousarray(W, np.float64)), arr)
    if st:
        raise ValueError(f"ref_output_checksums status {st}")
    return out


def ref_input_checksums(d: Dims, D, W):
    R_ = ref()
    cd1 = np.empty((d.C, d.H, d.H)); cd2 = np.empty_like(cd1)
    cw1 = np.empty((d.C, d.R, d.R)); cw2 = np.empty_like(cw1)
    st = R_.ref_input_checksums(C.byref(d), P(np.ascontiguousarray(D, np.float64)),
                                P(np.ascontiguousarray(W, np.float64)), P(cd1), P(cd2), P(cw1), P(cw2))
    if st:
        raise ValueError(f"ref_input_checksums status {st}")
    return cd1, cd2, cw1, cw2


def ref_output_summations(O, which, bias=None):
    R_ = ref()
    N, M, E, _ = O.shape
    out = [np.zeros(s) if which & (1 << k) else None for k, s in enumerate(_fam_shapes(N, M, E))]
    arr = (C.POINTER(C.c_double) * 7)(*[P(o) if o is not None else None for o in out])
    b = None if bias is None else np.ascontiguousarray(bias, np.float64)
    R_.ref_output_summations(N, M, E, P(np.ascontiguousarray(O, np.float64)), C.c_uint(which), P(b), arr)
    return out


def ref_protected_layer(d: Dims, D, W, bias, rc, clc, tau, O_conv=None, pre=None, want_output=False):
    R_ = ref()
    pre_arr, npre = _pre_array(pre)
    rep = Report()
    E = extent(d)
    Oout = np.zeros((d.N, d.M, E, E)) if want_output else None
    b = None if bias is None else np.ascontiguousarray(bias, np.float32)
    Oc = None if O_conv is None else np.ascontiguousarray(O_conv, np.float32)
    R_.ref_protected_layer_f64.argtypes = [
        C.POINTER(Dims), C.POINTER(C.c_float), C.POINTER(C.c_float), C.POINTER(C.c_float), C.c_int,
        C.c_int, C.c_double, C.POINTER(C.c_float), C.POINTER(PreFault), C.c_int, C.POINTER(Report),
        C.POINTER(C.c_double)]
    st = R_.ref_protected_layer_f64(C.byref(d), P(np.ascontiguousarray(D, np.float32), C.c_float),
                                    P(np.ascontiguousarray(W, np.float32), C.c_float), P(b, C.c_float),
                                    int(rc), int(clc), tau, P(Oc, C.c_float), pre_arr, npre,
                                    C.byref(rep), P(Oout))
    res = rep.as_dict()
    res["status"] = st
    if want_output:
        res["O"] = Oout
    return res


def ref_protected_layer_f32(d: Dims, D, W, bias=None, tau=1e-4):
    """The reference's shipped CPU path (T=float, default plan, direct conv)."""
    R_ = ref()
    rep = Report()
    E = extent(d)
    O = np.empty((d.N, d.M, E, E), np.float32)
    b = None if bias is None else np.ascontiguousarray(bias, np.float32)
    R_.ref_protected_layer_f32.argtypes = [C.POINTER(Dims), C.POINTER(C.c_float), C.POINTER(C.c_float),
                                           C.POINTER(C.c_float), C.c_double, C.POINTER(C.c_float),
                                           C.POINTER(Report)]
    st = R_.ref_protected_layer_f32(C.byref(d), P(np.ascontiguousarray(D, np.float32), C.c_float),
                                    P(np.ascontiguousarray(W, np.float32), C.c_float), P(b, C.c_float),
                                    tau, P(O, C.c_float), C.byref(rep))
    res = rep.as_dict()
    res["status"] = st
    return res, O


# ----------------------------------------------------------------------------- fault campaigns
class RefSpec(C.Structure):  # layout of ftc_fault_spec / ref_spec
    _fields_ = [("layer_index", C.c_int32), ("target", C.c_int32), ("checksum", C.c_int32), ("mode", C.c_int32),
                ("i", C.c_int64), ("j", C.c_int64), ("x", C.c_int64), ("y", C.c_int64), ("bit", C.c_uint32),
                ("pad_", C.c_uint32), ("seed", C.c_uint64)]


class RefTruth(C.Structure):
    _fields_ = [("benign", C.c_int32), ("expected_stage", C.c_int32), ("output_diverges", C.c_int32)]


class RefGrid(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("N", "M", "Ch", "H", "R")]


def ref_campaign(grids, n_runs, weights=(1, 1, 1, 1, 1, 1), seed=0):
    """The reference's campaign() (fault.hpp:195-271): list of (spec fields dict, truth dict)."""
    R_ = ref()
    g = (RefGrid * len(grids))(*[RefGrid(*x) for x in grids])
    specs = (RefSpec * max(1, n_runs))()
    truths = (RefTruth * max(1, n_runs))()
    w = (C.c_double * 6)(*weights)
    R_.ref_campaign.argtypes = [C.POINTER(RefGrid), C.c_int, C.c_longlong, C.POINTER(C.c_double), C.c_uint64,
                                C.POINTER(RefSpec), C.POINTER(RefTruth)]
    code = R_.ref_campaign(g, len(grids), n_runs, w, seed, specs, truths)
    if code:
        raise RuntimeError(f"ref_campaign failed ({code})")
    out = []
    for r in range(n_runs):
        s, t = specs[r], truths[r]
        out.append(({k: getattr(s, k) for k, _ in RefSpec._fields_ if k != "pad_"},
                    {k: getattr(t, k) for k, _ in RefTruth._fields_}))
    return out


def ref_apply_spec(spec: dict, N, C_, H, M, R, E, D=None, W=None, O=None, cd1=None, cd2=None, cw1=None, cw2=None):
    """make_hooks(f) of the reference applied to copies of the given host tensors (float
    D/W/O; FP64 checksums); returns the perturbed copies in the same order."""
    R_ = ref()
    s = RefSpec(**spec)
    cp = [None if a is None else np.ascontiguousarray(a).copy() for a in (D, W, O)]
    ck = [None if a is None else np.ascontiguousarray(a, np.float64).copy() for a in (cd1, cd2, cw1, cw2)]
    fp = lambda a: None if a is None else a.ctypes.data_as(C.POINTER(C.c_float))
    dp = lambda a: None if a is None else a.ctypes.data_as(C.POINTER(C.c_double))
    R_.ref_apply_spec.argtypes = [C.POINTER(RefSpec)] + [C.c_int] * 6 + [C.POINTER(C.c_float)] * 3 + \
        [C.POINTER(C.c_double)] * 4
    code = R_.ref_apply_spec(C.byref(s), N, C_, H, M, R, E, *[fp(a) for a in cp], *[dp(a) for a in ck])
    if code:
        raise RuntimeError(f"ref_apply_spec failed ({code})")
    return cp + ck


def ref_plan_to_json(plans: dict) -> str:
    """The reference's plan_to_json (serialize.cpp:115-124); plans: name -> dict with
    rc_enabled, clc_enabled, tau, t0, t1, t2, p_r."""
    R_ = ref()
    names = list(plans)
    arr_n = (C.c_char_p * max(1, len(names)))(*[n.encode() for n in names])
    vals = []
    for n in names:
        p = plans[n]
        vals += [float(p["rc_enabled"]), float(p["clc_enabled"]), p["tau"], p["t0"], p["t1"], p["t2"], p["p_r"]]
    v = (C.c_double * max(1, len(vals)))(*vals)
    buf = C.create_string_buffer(1 << 20)
    R_.ref_plan_to_json.argtypes = [C.c_int, C.POINTER(C.c_char_p), C.POINTER(C.c_double), C.c_char_p, C.c_longlong]
    R_.ref_plan_to_json.restype = C.c_longlong
    n = R_.ref_plan_to_json(len(names), arr_n, v, buf, len(buf))
    if n < 0:
        raise RuntimeError("ref_plan_to_json failed")
    return buf.value.decode()


def ref_corpus_to_jsonl(entries) -> str:
    """The reference's corpus_to_jsonl (serialize.cpp:68-80); entries: (spec dict, truth dict)."""
    R_ = ref()
    specs = (RefSpec * max(1, len(entries)))(*[RefSpec(**s) for s, _ in entries])
    truths = (RefTruth * max(1, len(entries)))(*[RefTruth(**t) for _, t in entries])
    buf = C.create_string_buffer(1 << 22)
    R_.ref_corpus_to_jsonl.argtypes = [C.c_int, C.POINTER(RefSpec), C.POINTER(RefTruth), C.c_char_p, C.c_longlong]
    R_.ref_corpus_to_jsonl.restype = C.c_longlong
    n = R_.ref_corpus_to_jsonl(len(entries), specs, truths, buf, len(buf))
    if n < 0:
        raise RuntimeError("ref_corpus_to_jsonl failed")
    return buf.value.decode()


# ----------------------------------------------------------------------------- model files / reports
STAGE_CODES = {"none": 0, "reload": 1, "coc": 2, "rc": 3, "clc": 4, "fc": 5, "discard": 6, "recompute": 7}  # report.hpp:12-21


def ref_parse_model_config(text: str) -> int:
    """parse_model_config status through the reference: 0 ok, 2 ConfigError, 1 ShapeError."""
    L = ref()
    L.ref_parse_model_config.argtypes = [C.c_char_p, C.POINTER(C.c_int)]
    n = C.c_int(0)
    return L.ref_parse_model_config(text.encode(), C.byref(n))


def ref_make_weights(config_text: str, seed: int, path: str) -> int:
    L = ref()
    L.ref_make_weights.argtypes = [C.c_char_p, C.c_uint64, C.c_char_p]
    return L.ref_make_weights(config_text.encode(), C.c_uint64(seed), path.encode())


def ref_load_weights(config_text: str, path: str) -> int:
    L = ref()
    L.ref_load_weights.argtypes = [C.c_char_p, C.c_char_p]
    return L.ref_load_weights(config_text.encode(), path.encode())


def ref_report_to_json(reports, timings=False, campaign=None) -> str:
    """report_to_json (serialize.cpp:174-193) of LayerReport-like objects through the
    reference; campaign = (runs, detected, above, recovered, mismatches, fatals) wraps
    them as a CampaignReport."""
    L = ref()
    n = len(reports)
    names = (C.c_char_p * max(1, n))(*[r.layer.encode() for r in reports])
    ints, blocks, stages, tkeys, tvals = [], [], [], [], []
    for r in reports:
        ints += [int(r.detected), STAGE_CODES[r.stage], int(r.weights_reloaded), int(r.recomputed),
                 len(r.corrected_blocks), len(r.stages_attempted), len(r.timings), 0]
        for b in r.corrected_blocks:
            blocks += [int(b[0]), int(b[1])]
        stages += [STAGE_CODES[s] for s in r.stages_attempted]
        for k in sorted(r.timings):
            tkeys.append(k.encode())
            tvals.append(float(r.timings[k]))
    ia = (C.c_int * max(1, len(ints)))(*ints)
    ba = (C.c_longlong * max(1, len(blocks)))(*blocks)
    sa = (C.c_int * max(1, len(stages)))(*stages)
    ka = (C.c_char_p * max(1, len(tkeys)))(*tkeys)
    va = (C.c_double * max(1, len(tvals)))(*tvals)
    camp = (C.c_longlong * 7)(*(list(campaign or (0,) * 6) + [0]))
    cap = 1 << 22
    out = C.create_string_buffer(cap)
    L.ref_report_to_json.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_char_p, C.c_longlong]
    L.ref_report_to_json.restype = C.c_longlong
    k = L.ref_report_to_json(n, names, ia, ba, sa, ka, va, int(bool(timings)), int(campaign is not None), camp, out,
                             cap)
    if k < 0:
        raise RuntimeError("ref_report_to_json failed")
    return out.raw[:k].decode()


# ----------------------------------------------------------------------------- back-propagation
class _GradHook(C.Structure):
    _fields_ = [("target", C.c_int), ("index", C.c_longlong), ("mode", C.c_int), ("value", C.c_double)]


def _hooks(hooks):
    """hooks: iterable of (target 'dW'|'dD', flat index, mode 'set'|'add', value)"""
    hooks = list(hooks or ())
    arr = (_GradHook * max(1, len(hooks)))(*[_GradHook(0 if t == "dW" else 1, int(i), 0 if m == "set" else 1,
                                                       float(v)) for t, i, m, v in hooks])
    return arr, len(hooks)


def _bwd_shapes(d: Dims):
    E = extent(d)
    return (d.M, d.C, d.R, d.R), (d.N, d.C, d.H, d.H), (d.N, d.M, E, E)


def conv_backward(d: Dims, D, W, dO, lib=None):
    """conv_backward<double> (conv.hpp:150-185): oracle restatement, or the reference
    itself with lib=ref()."""
    sw, sd, _ = _bwd_shapes(d)
    dW, dD = np.empty(sw), np.empty(sd)
    L = lib or oracle()
    fn = L.or_conv_backward_f64 if L is oracle() else L.ref_conv_backward
    fn.argtypes = [C.POINTER(Dims)] + [C.c_void_p] * 5
    st = fn(C.byref(d), P(_f64(D)), P(_f64(W)), P(_f64(dO)), P(dW), P(dD))
    return st, dW, dD


def protected_backward(d: Dims, D, W, dO, tau, hooks=(), lib=None):
    """run_protected_backward<double> (workflow.hpp:350-417) -> (status, dW, dD,
    {dw_detected, dd_detected, recomputed})"""
    sw, sd, _ = _bwd_shapes(d)
    dW, dD = np.empty(sw), np.empty(sd)
    arr, n = _hooks(hooks)
    L = lib or oracle()
    if L is oracle():
        f = (C.c_int * 3)()
        L.or_protected_backward.argtypes = [C.POINTER(Dims)] + [C.c_void_p] * 3 + [C.c_double, C.c_void_p, C.c_int,
                                                                                   C.c_void_p, C.c_void_p,
                                                                                   C.c_void_p, C.c_void_p,
                                                                                   C.c_void_p]
        st = L.or_protected_backward(C.byref(d), P(_f64(D)), P(_f64(W)), P(_f64(dO)), tau, arr, n, P(dW), P(dD),
                                     C.byref(f, 0), C.byref(f, 4), C.byref(f, 8))
    else:
        f = (C.c_int * 3)()
        L.ref_protected_backward.argtypes = [C.POINTER(Dims)] + [C.c_void_p] * 3 + [C.c_double, C.c_void_p, C.c_int,
                                                                                    C.c_void_p, C.c_void_p,
                                                                                    C.c_void_p]
        st = L.ref_protected_backward(C.byref(d), P(_f64(D)), P(_f64(W)), P(_f64(dO)), tau, arr, n, P(dW), P(dD),
                                      f)
    return st, dW, dD, {"dw_detected": bool(f[0]), "dd_detected": bool(f[1]), "recomputed": bool(f[2])}
