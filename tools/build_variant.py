"""Build variants/<name>/libdsg_b200.so with extra nvcc defines for one
source (the others reuse the in-tree objects); select at run time with
DSG_B200_LIB=variants/<name>/libdsg_b200.so.

    python tools/build_variant.py NAME SOURCE.cu -DMACRO=VALUE ...
"""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2006_16423_b200 import _build as B

name, src, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
out = os.path.join(ROOT, os.environ.get("DSG_VARIANT_DIR", "variants"), name)
os.makedirs(out, exist_ok=True)
obj = os.path.join(out, src.replace(".cu", ".o"))
subprocess.run([B.nvcc(), *B.NVCC_FLAGS, *defs, "-I", os.path.join(ROOT, "include"), "-I", B.CSRC,
                "-c", os.path.join(B.CSRC, src), "-o", obj], check=True)
objs = [obj if s == src else os.path.join(B.HERE, "build", s.replace(".cu", ".o")) for s in B.SOURCES]
subprocess.run([B.nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o",
                os.path.join(out, "libdsg_b200.so")], check=True)
print(os.path.join(out, "libdsg_b200.so"))
