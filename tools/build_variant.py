"""Build a variant of libtpla.so with extra nvcc defines, for A/B timing on the GPU box:
    python tools/build_variant.py NAME -DTPLA_POLY_MASK=0xAA ...   ->  build/variants/libtpla_NAME.so
then run with TPLA_LIB=build/variants/libtpla_NAME.so.  Only the sources are recompiled."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_15881_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out_dir = os.path.join(B.ROOT, "build", "variants", name)
os.makedirs(out_dir, exist_ok=True)
objs = []
for src in B.sources():
    obj = os.path.join(out_dir, os.path.basename(src) + ".o")
    r = subprocess.run([B.NVCC, "-c", src, "-o", obj] + B.flags() + defs, capture_output=True, text=True)
    if r.returncode:
        sys.exit(r.stderr)
    objs.append(obj)
lib = os.path.join(B.ROOT, "build", "variants", f"libtpla_{name}.so")
r = subprocess.run([B.NVCC, "-shared", "-o", lib] + objs + B.ARCH + ["-ldl", "-Xcompiler", "-fPIC"],
                   capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr)
print(lib)
