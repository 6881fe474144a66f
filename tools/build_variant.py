"""Experiments: build the library with one source file swapped (or a -D flag) into
build/variants/<name>.so; select it at run time with FTC_LIB_PATH."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2003_12203_b200 import build as B  # noqa: E402


def main(name, swap_src=None, swap_with=None, extra=()):
    out_dir = os.path.join(ROOT, "build", "variants", name)
    os.makedirs(out_dir, exist_ok=True)
    objs = []
    for src in B._sources():
        use = swap_with if (swap_src and os.path.basename(src) == swap_src) else src
        obj = os.path.join(out_dir, os.path.basename(src) + ".o")
        cmd = [B.NVCC, *B.ARCH, *B.FLAGS, "-I" + B.CSRC, *extra, "-c", use, "-o", obj]
        subprocess.run(cmd, check=True, capture_output=True)
        objs.append(obj)
    lib = os.path.join(ROOT, "build", "variants", name + ".so")
    subprocess.run([B.NVCC, *B.ARCH, "-shared", "-cudart", "static", "-o", lib, *objs], check=True)
    print(lib)


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0], a[1] if len(a) > 1 and a[1] != "-" else None, a[2] if len(a) > 2 else None, a[3:])
