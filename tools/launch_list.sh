#!/bin/bash
# ncu launch list (per-kernel durations, cold and serialised) of warm solves:
#   gpurun -- bash tools/launch_list.sh C2 tag
W=${1:-C2}; TAG=${2:-ll}
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_${W//[:,@]/_}.csv python tools/profile_one.py "$W" 2 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/${TAG}_${W//[:,@]/_}.csv 2
