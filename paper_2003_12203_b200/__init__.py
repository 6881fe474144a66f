"""B200-native ABFT-protected convolution (FT-CNN, arXiv 2003.12203).

The hot path -- input/filter checksums, the conv, fused output summations, CoC-D
detection and the CoC/RC/ClC/FC locate-correct-recompute workflow -- runs in
hand-written sm_100a CUDA kernels behind the C ABI in include/ftc_abi.h
(libftconv_b200.so).  This Python package is a thin ctypes mirror of the
reference's C++ API (proj/core/include/ftconv/) used by tests and bench.py.
"""
from .ftconv import (  # noqa: F401
    BackwardReport, GradFault, conv_backward, run_protected_backward,
    ConfigError, ConvParams, Fault, IntegrityError, IoError, LayerPlan, LayerReport,
    ProtectedConv, ShapeError, conv_forward, detect_coc_d, input_checksums, output_bitflip,
    output_checksums, output_extent, output_summations, run_protected_layer, set_conv_engine,
    verify_kernel,
)

__all__ = [
    "BackwardReport", "GradFault", "conv_backward", "run_protected_backward",
    "ConfigError", "ConvParams", "Fault", "IntegrityError", "IoError", "LayerPlan", "LayerReport",
    "ProtectedConv", "ShapeError", "conv_forward", "detect_coc_d", "input_checksums",
    "output_bitflip", "output_checksums", "output_extent", "output_summations",
    "run_protected_layer", "set_conv_engine", "verify_kernel",
]
