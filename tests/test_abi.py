"""CPU-side checks of the C-ABI boundary: the CUDA library loads, exports
every entry point include/dsg_b200.h declares, and refuses to compute
without a GPU (no CPU fallback)."""
import ctypes as C
import os
import re

import pytest

from paper_2006_16423_b200 import _abi, solver
from paper_2006_16423_b200.errors import DeviceError
from paper_2006_16423_b200.graph import DeviceConfig
from paper_2006_16423_b200.workloads import diamond4

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    text = open(os.path.join(ROOT, "include", "dsg_b200.h")).read()
    return sorted(set(re.findall(r"\b(dsg_[a-z_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("dsg_dp_solve", "dsg_result_free", "dsg_enumerate_ideals", "dsg_ideals_free",
                     "dsg_default_options", "dsg_version", "dsg_device_count",
                     "dsg_kernel_launch_count"):
        assert required in names


def test_library_exports_every_declared_symbol():
    lib = solver.load_library()
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_struct_sizes_match_the_header_layout():
    # pointer-bearing structs are laid out as in dsg_b200.h (x86-64 LP64)
    assert C.sizeof(_abi.dsg_rat) == 16
    assert C.sizeof(_abi.dsg_graph) == 4 + 4 + 8 * 7 + 4 + 4 + 16 + 4 + 4 + 16
    assert C.sizeof(_abi.dsg_options) == 32
    assert C.sizeof(_abi.dsg_block) == 24


def test_version_string():
    lib = solver.load_library()
    assert b"sm_100a" in lib.dsg_version()


def test_default_options_match_reference_budget():
    lib = solver.load_library()
    o = _abi.dsg_options()
    lib.dsg_default_options(C.byref(o))
    assert o.ideal_budget == 5_000_000  # kDefaultIdealBudget, graph.hpp:251
    assert o.device == -1


@pytest.mark.skipif(solver.load_library().dsg_device_count() > 0, reason="GPU present")
def test_no_cpu_fallback_without_a_gpu():
    with pytest.raises(DeviceError):
        solver.solve_maxload_inference(diamond4(), DeviceConfig(2, 0, 4))


def test_sass_is_sm100a():
    """The shipped library carries sm_100a SASS (cuobjdump), not PTX-only."""
    import shutil
    import subprocess
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "--list-elf", solver.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
