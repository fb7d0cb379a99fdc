#!/bin/bash
# Quick GPU iteration: parity tests, per-workload device times, optional traces.
#   tools/gpu_quick.sh [tests|notests] [trace]
mkdir -p gpurun_out
if [ "${1:-tests}" = tests ]; then
  timeout 600 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/q_tests.log 2>&1
  echo "TESTS_EXIT=$?" >> gpurun_out/q_tests.log
  tail -3 gpurun_out/q_tests.log
fi
for w in ${WORKLOADS:-C1 C2 C3 C4}; do
  timeout 60 python tools/profile_one.py $w 5 2>&1 | tail -1
done | tee gpurun_out/q_times.log
if [ "${2:-}" = trace ]; then
  for w in ${TRACE_WL:-C2 C4}; do
    DSG_TRACE_FILE=/tmp/trace_$w.bin timeout 120 python tools/profile_one.py $w 3 > gpurun_out/qtrace_$w.log 2>&1
    python tools/trace_view.py /tmp/trace_$w.bin 1 >> gpurun_out/qtrace_$w.log 2>&1
  done
fi
