#!/bin/bash
# ncu --set full capture (with source) of the enumeration kernel of a workload:
#   gpurun -- bash tools/ncu_enum.sh C4 tag
W=${1:-C4}
TAG=${2:-enum}
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:enumerate_levels -s 2 -c 1 \
  -o gpurun_out/${TAG} python tools/profile_one.py "$W" 3 > gpurun_out/${TAG}_ncu.log 2>&1
echo "NCU_EXIT=$?" >> gpurun_out/${TAG}_ncu.log
tail -2 gpurun_out/${TAG}_ncu.log
