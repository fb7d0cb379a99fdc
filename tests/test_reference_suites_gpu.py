"""The reference's OWN test programs, run against the B200 drop-in.

integration/Makefile compiles /root/reference/proj/tests/{acceptance.cpp,
test_*.cpp} unmodified and links them with integration/dp_solver_b200.cpp
(which replaces src/dp_solver.cpp and src/ideals.cpp by calls into
libdsg_b200.so).  build() produces the binaries in the build container; they
travel to the GPU box with the snapshot.  Every solve_maxload_* and
enumerate_ideals* call in those suites therefore runs on the B200.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "integration", "_build")

pytestmark = pytest.mark.gpu


def _run(name, *args):
    exe = os.path.join(BUILD, name)
    if not os.path.exists(exe):
        pytest.skip(f"{name} not built (make -C integration needs /root/reference)")
    p = subprocess.run([exe, *args], capture_output=True, text=True, timeout=600, cwd=BUILD)
    return p.returncode, p.stdout + p.stderr


@pytest.mark.parametrize("suite", ["rational", "graph_core", "ingest", "preprocess", "dp_solver",
                                   "ip_builder", "baselines", "pipeline_sim"])
def test_reference_unit_suite_on_b200(gpu, suite):
    rc, out = _run("unit_b200", f"-ts={suite}")
    assert rc == 0, out[-3000:]
    assert " 0 failed" in out


def test_reference_acceptance_on_b200(gpu):
    rc, out = _run("acceptance_b200")
    assert rc == 0, out[-3000:]
    for ac in ("AC-1", "AC-2", "AC-3", "AC-4", "AC-5", "AC-6", "AC-8", "AC-9"):
        line = next(l for l in out.splitlines() if l.startswith(ac))
        assert "[PASS]" in line, line
