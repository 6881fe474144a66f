"""The C++ host API (include/ftconv_b200/ftconv.hpp) over the C ABI, driven like the
reference's own doctest units (tests/cpp/test_api.cpp)."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_cpp_api_program(tmp_path):
    from paper_2003_12203_b200.build import build
    lib = build()
    exe = tmp_path / "test_api"
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_api.cpp"), "-o", str(exe),
                    lib, f"-Wl,-rpath,{os.path.dirname(lib)}"], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
