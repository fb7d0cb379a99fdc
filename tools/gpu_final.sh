#!/bin/bash
# Round-end evidence in one call: full GPU suite, smoke, bench lines for every
# config + the reference arm, the C2 launch list and one full ncu capture.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/final_tests.log 2>&1
echo "TESTS_EXIT=$?" >> gpurun_out/final_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1
echo "SMOKE_EXIT=$?" >> gpurun_out/final_smoke.log
bash tools/gpu_profile_round.sh
