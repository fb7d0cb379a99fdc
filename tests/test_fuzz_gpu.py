"""Randomised parity against the oracle port (tools/fuzz_parity.py): module
chains of 60-900 nodes (ragged and wide word counts), K in 1..16, L in 0..4,
inference and mirrored training, binding and loose memory limits."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [3, 29])
def test_random_module_chains_match_oracle(gpu, seed):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "fuzz_parity.py"), "30", str(seed)],
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
