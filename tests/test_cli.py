"""§8(f) row 2: the reference's own command line (tools/dagsplit_main.cpp,
compiled unchanged against integration/cli_shim/CLI11.hpp) on the B200
drop-in.  `solve --solver dp|dpl` must write the same result JSON as the
same CLI on the CPU reference outside wallTimeSeconds and the tie-broken
assignment: same objective, status and device labels, every node
assigned, worst load == objective (the partition is verified, not compared:
SURVEY 8(c)).  Reruns are byte-identical (cli_smoke.sh:39-46) and the exit
codes stay 2/3/4 (dagsplit_main.cpp:338-365)."""
import json
import os

import pytest

from cli_io import CLI_B200, CLI_REF, run_cli, strip_wall, workload_json
from paper_2006_16423_b200 import workloads as wl
from paper_2006_16423_b200.graph import DeviceConfig

needs_cli = pytest.mark.skipif(not (os.path.exists(CLI_B200) and os.path.exists(CLI_REF)),
                               reason="integration/_build CLIs not built (make -C integration)")

D4 = (wl.diamond4(), DeviceConfig(2, 1, 4))
D4T = (wl.mirror_training(wl.diamond4()), DeviceConfig(2, 0, 8))
TOO_BIG = '{"devices":{"accelerators":1,"cpus":0,"memoryLimit":1},' \
          '"nodes":[{"id":1,"cpuTime":1,"accTime":1,"commTime":0,"memory":5}],"edges":[]}'


def _cases():
    out = [("d4", *D4), ("d4_training", *D4T)]
    for s in (3, 11, 42):
        inst = wl.random_instance(s)
        out.append((f"random{s}", inst.graph, inst.config))
    out.append(("C1", wl.standin("C1").graph, wl.standin("C1").config))
    return out


def _write(tmp_path, name, text):
    p = tmp_path / f"{name}.json"
    p.write_text(text)
    return p


@needs_cli
def test_reference_cli_through_shim(tmp_path):
    """The checker side: the CPU-reference CLI parses and solves via the shim."""
    w = _write(tmp_path, "d4", workload_json(*D4))
    r = run_cli(CLI_REF, "solve", w, "--solver", "dp", "-o", tmp_path / "o.json")
    assert r.returncode == 0, r.stderr
    assert json.loads((tmp_path / "o.json").read_text())["objectiveValue"] == 6.0
    assert run_cli(CLI_REF).returncode == 109           # subcommand required
    assert run_cli(CLI_REF, "solve").returncode == 106  # input required


@pytest.mark.gpu
@needs_cli
@pytest.mark.parametrize("solver_args", [["--solver", "dp"], ["--solver", "dpl", "--seed", "1"]],
                         ids=["dp", "dpl"])
@pytest.mark.parametrize("case", _cases(), ids=[c[0] for c in _cases()])
def test_cli_result_json_identical_to_reference(gpu, tmp_path, case, solver_args):
    name, g, cfg = case
    w = _write(tmp_path, name, workload_json(g, cfg))
    outs = []
    for binary in (CLI_B200, CLI_REF):
        o = tmp_path / f"{name}_{os.path.basename(binary)}.json"
        r = run_cli(binary, "solve", w, *solver_args, "-o", o)
        assert r.returncode == 0, r.stderr
        outs.append(json.loads(o.read_text()))
    ours, ref = outs
    for key in ("objective", "objectiveValue", "status", "solver"):
        assert ours[key] == ref[key], key
    # fewest devices (dp_solver.cpp:337-351) is tie-free: same labels used
    assert sorted(ours["perDeviceLoads"]) == sorted(ref["perDeviceLoads"])
    assert max(ours["perDeviceLoads"].values()) == ours["objectiveValue"]
    assert sorted(a["nodeId"] for a in ours["assignment"]) == sorted(n.id for n in g.nodes())


@pytest.mark.gpu
@needs_cli
def test_cli_exit_codes_and_rerun(gpu, tmp_path):
    w = _write(tmp_path, "d4", workload_json(*D4))
    a, b = tmp_path / "a.json", tmp_path / "b.json"
    assert run_cli(CLI_B200, "solve", w, "--solver", "dp", "-o", a).returncode == 0
    assert run_cli(CLI_B200, "solve", w, "--solver", "dp", "-o", b).returncode == 0
    assert strip_wall(a.read_text()) == strip_wall(b.read_text())
    assert '"objectiveValue": 6.0' in a.read_text()
    broken = _write(tmp_path, "broken", '{"broken')
    assert run_cli(CLI_B200, "solve", broken).returncode == 2
    assert run_cli(CLI_B200, "solve", _write(tmp_path, "big", TOO_BIG)).returncode == 3
    assert run_cli(CLI_B200, "solve", w, "--ideal-budget", 2).returncode == 4
    t = _write(tmp_path, "d4t", workload_json(*D4T))
    assert run_cli(CLI_B200, "solve", t, "--solver", "dp", "-o", tmp_path / "t.json").returncode == 0
