#!/bin/bash
# Where the nested pairs go (diagnostic build var/stats, -DDSG_PAIR_STATS):
#   gpurun -- bash tools/pair_stats.sh
mkdir -p gpurun_out
for w in C2 C3 C4 C1 C5:8,2,7,600 C5:16,1,1,300 C2@seed2 C2@D1000; do
  echo "== $w"
  DSG_B200_LIB=var/stats/libdsg_b200.so python tools/profile_one.py "$w" 1 2>&1 | grep -E "DSG_PAIR_STATS|obj|pairs" | tail -2
done
