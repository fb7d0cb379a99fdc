#!/bin/bash
# One ncu --set full capture (with source) of the dataflow DP kernel of a
# workload, with an nvidia-smi clock record taken while ncu runs.
#   gpurun -- bash tools/ncu_capture.sh C2 r2_c2
W=${1:-C2}
TAG=${2:-cap}
mkdir -p gpurun_out
nvidia-smi --query-gpu=timestamp,clocks.sm,clocks.max.sm,clocks.mem,power.draw,temperature.gpu,clocks_event_reasons.active \
  --format=csv -lms 200 > gpurun_out/${TAG}_clocks.csv 2>&1 &
SMI=$!
timeout 900 ncu --set full --import-source on --clock-control none -k regex:persistent_levels -s 2 -c 1 \
  -o gpurun_out/${TAG} python tools/profile_one.py "$W" 3 > gpurun_out/${TAG}_ncu.log 2>&1
echo "NCU_EXIT=$?" >> gpurun_out/${TAG}_ncu.log
kill $SMI
tail -2 gpurun_out/${TAG}_ncu.log
