"""CPU checks of the drop-in boundary: the C-ABI library builds, loads without a GPU
and exports every symbol include/ftc_abi.h declares; host-side logic of the
Python mirror (no compute calls)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def _declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "ftc_abi.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(ftc_[a-z0-9_]+)\s*\(", hdr)))


def test_header_declares_the_expected_abi():
    from paper_2003_12203_b200 import _abi
    assert sorted(_abi.EXPORTS) == _declared_symbols()


def test_library_loads_and_exports_every_declared_symbol():
    from paper_2003_12203_b200 import _abi
    from paper_2003_12203_b200.build import build
    build()
    lib = C.CDLL(_abi.LIB_PATH)
    for sym in _declared_symbols():
        assert hasattr(lib, sym), sym
    assert lib.ftc_abi_version() == 1


def test_extent_rule_without_gpu():
    """tensor.hpp:100-107 through the ABI (pure host logic)."""
    from paper_2003_12203_b200 import ConfigError, ConvParams, output_extent
    assert output_extent(56, 3, ConvParams(pad=1)) == 56
    assert output_extent(227, 11, ConvParams(stride=4)) == 55
    with pytest.raises(ConfigError):
        output_extent(8, 3, ConvParams(stride=2))
    with pytest.raises(ConfigError):
        output_extent(2, 3, ConvParams())


def test_fault_struct_layout_matches_header():
    from paper_2003_12203_b200 import _abi
    assert C.sizeof(_abi.Fault) == 48
    assert C.sizeof(_abi.ConvDesc) == 36
    assert C.sizeof(_abi.Plan) == 48


def test_synth_generators_are_deterministic():
    from paper_2003_12203_b200 import synth
    a, b = synth.config1(7), synth.config1(7)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    D = a[0]
    assert abs((D == 0).mean() - 0.5) < 0.01 and D.max() <= 1.0
    assert abs(a[1].std() - np.sqrt(2 / 576)) < 0.002
    s = [synth.flip_sample(99, r, 16, 64, 56) for r in range(200)]
    assert all(20 <= t[4] <= 30 for t in s) and len(set(s)) > 190
