"""In-tree build of libdsg_b200.so (sm_100a) and the test-only oracle libraries.

    python -m paper_2006_16423_b200._build          # product library
    python -m paper_2006_16423_b200._build --all    # + oracle/_build, oracle/_ref

The .so lands next to this file so it travels to the GPU box with the
snapshot (git-ignored, not gpurun-ignored).  nvcc cross-compiles for sm_100a
without a GPU.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libdsg_b200.so")
SOURCES = ["capi.cu", "enumerate.cu", "describe.cu", "transition.cu", "persistent.cu",
           # the dataflow kernel's variants, one translation unit each (parallel nvcc)
           "persistent_x_i32_inf.cu", "persistent_x_i32_train.cu",
           "persistent_g_i32_inf.cu", "persistent_g_i32_train.cu",
           "persistent_g_i64_inf.cu", "persistent_g_i64_train.cu"]
HEADERS = ["dsg_device.cuh", "dsg_internal.h", "scan.cuh", "persistent_impl.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "--expt-relaxed-constexpr", "--extended-lambda",
    "-Xcompiler", "-fPIC,-O3",
    "-Xptxas", "-warn-spills",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_lib(force: bool = False, verbose: bool = False, extra=()) -> str:
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "dsg_b200.h"))
    if not force and not _stale(LIB, deps):
        return LIB
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    hdrs = [d for d in deps if not d.endswith(".cu")]
    for s in SOURCES:
        obj = os.path.join(objdir, s.replace(".cu", ".o"))
        objs.append(obj)
        if not force and not extra and not _stale(obj, [os.path.join(CSRC, s), *hdrs]):
            continue  # object newer than its source and every header
        cmd = [nvcc(), *NVCC_FLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-I", CSRC,
               "-c", os.path.join(CSRC, s), "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append((s, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    failed = []
    for s, p in procs:
        out, _ = p.communicate()
        text = out.decode(errors="replace")
        if p.returncode != 0:
            failed.append(f"--- {s}\n{text}")
        elif verbose and text.strip():
            print(text)
    if failed:
        raise RuntimeError("nvcc failed:\n" + "\n".join(failed))
    link = [nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", LIB]
    subprocess.run(link, check=True)
    return LIB


def build_oracle(ref: bool = True) -> None:
    """Test infrastructure: oracle/_build (C restatement) and, where the
    reference sources exist (this container), oracle/_ref."""
    jobs = str(os.cpu_count() or 4)
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "-j", jobs, "all"], check=True)
    if ref and os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "-j", jobs, "ref"], check=True)
        # the reference's own test programs linked against the B200 drop-in
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "integration"), "-j", jobs], check=True)


if __name__ == "__main__":
    force = "--force" in sys.argv
    print(build_lib(force=force, verbose="-v" in sys.argv))
    if "--all" in sys.argv:
        build_oracle()
