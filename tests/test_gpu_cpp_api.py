"""The C++ host API (include/ftconv_b200/*.hpp) over the C ABI, driven like the
reference's own doctest units: tests/cpp/test_api.cpp (conv / run_protected_layer /
backward), tests/cpp/test_blocks.cpp (the checksum and detection building blocks,
bitwise against host restatements at T=double) and tests/cpp/test_stack.cpp (a conv
stack through the fused clean path vs the single-layer host API)."""
import os
import subprocess

import pytest

from conftest import ROOT

PROGRAMS = ("test_api", "test_blocks", "test_stack")


def _compile(src, out, lib=None, syntax_only=False):
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"), src]
    if syntax_only:
        cmd += ["-fsyntax-only"]
    else:
        cmd += ["-o", str(out), lib, f"-Wl,-rpath,{os.path.dirname(lib)}"]
    subprocess.run(cmd, check=True)


@pytest.mark.parametrize("prog", PROGRAMS)
def test_cpp_program_compiles(prog):
    """CPU: every C++ test program compiles against the headers alone."""
    _compile(os.path.join(ROOT, "tests", "cpp", prog + ".cpp"), None, syntax_only=True)


@pytest.mark.gpu
@pytest.mark.parametrize("prog", PROGRAMS)
def test_cpp_program_runs(prog, tmp_path):
    from paper_2003_12203_b200.build import build
    lib = build()
    exe = tmp_path / prog
    _compile(os.path.join(ROOT, "tests", "cpp", prog + ".cpp"), exe, lib)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
