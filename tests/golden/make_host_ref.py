"""Fold the full-size reference solves timed on the GPU box's host
(tools/cpu_ref_host.sh -> profiles/r2_cpu_ref_host/*.json: the UNMODIFIED
reference, oracle/_ref, one solve per workload) into a golden file of
objectives the device path must reproduce: tests/golden/host_reference.json.

    python tests/golden/make_host_ref.py
"""
import glob
import json
import os

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))

rows = []
for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r2_cpu_ref_host", "*.json"))):
    for r in json.load(open(path)):
        rows.append({k: r[k] for k in ("workload", "name", "nodes", "ideals", "pairs_closed_form",
                                       "k", "l", "objective", "ref_wall_s", "us_per_pair")})
rows.sort(key=lambda r: r["pairs_closed_form"])
with open(os.path.join(HERE, "host_reference.json"), "w") as f:
    json.dump(rows, f, indent=1)
print(len(rows), "rows")
