#!/bin/bash
# Quick GPU iteration: selected pytest files, then bench lines for the given
# workloads (device + e2e, no CPU baseline).  Usage:
#   gpurun -- bash tools/gpu_check.sh "tests/test_a.py tests/test_b.py" "C2 C4 C1"
mkdir -p gpurun_out
TESTS=${1:-}
WLS=${2:-C2}
TAG=${3:-chk}
if [ -n "$TESTS" ]; then
  timeout 1500 python -m pytest $TESTS -m gpu -q -x > gpurun_out/${TAG}_tests.log 2>&1
  echo "TESTS_EXIT=$?" >> gpurun_out/${TAG}_tests.log
  tail -3 gpurun_out/${TAG}_tests.log
fi
for w in $WLS; do
  timeout 300 python bench.py --workload "$w" --steps 10 --warmup 3 --no-cpu-baseline \
    > gpurun_out/${TAG}_bench_${w//[:,@]/_}.json 2> gpurun_out/${TAG}_bench_${w//[:,@]/_}.err
  python - "$w" gpurun_out/${TAG}_bench_${w//[:,@]/_}.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(sys.argv[1], "dev_ms %.3f" % d["ms_per_step"], "kern_ms %.3f" % d["roofline"]["kernel_ms_per_step"],
          "e2e_ms %.3f" % d["e2e"]["ms_per_step"], "clk", d["clocks"].get("sm_mhz"), d["clocks"].get("reasons"))
except Exception as e:
    print(sys.argv[1], "bench failed", e)
PY
done
