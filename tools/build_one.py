"""Recompile one csrc/*.cu object and relink libdsg_b200.so (dev loop).

    python tools/build_one.py enumerate.cu [more.cu ...]
"""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_16423_b200 import _build as B

objdir = os.path.join(B.HERE, "build")
for s in sys.argv[1:]:
    obj = os.path.join(objdir, s.replace(".cu", ".o"))
    subprocess.run([B.nvcc(), *B.NVCC_FLAGS, "-I", os.path.join(B.ROOT, "include"), "-I", B.CSRC,
                    "-c", os.path.join(B.CSRC, s), "-o", obj], check=True)
objs = [os.path.join(objdir, s.replace(".cu", ".o")) for s in B.SOURCES]
subprocess.run([B.nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", B.LIB],
               check=True)
print(B.LIB)
