#!/bin/bash
# Device ms of a workload under environment knob settings:
#   gpurun -- bash tools/knob_bench.sh C3 "DSG_DEAD_SKIP=0" "DSG_COVER_FIN=0" ...
W=$1; shift
mkdir -p gpurun_out
for kv in "" "$@"; do
  env $kv python tools/knob_time.py "$W" 15 2>&1 | tail -1 | sed "s/^/[$kv] /"
done
