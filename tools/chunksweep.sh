#!/bin/bash
# DP kernel time vs. recent-level chunking (DSG_RECENT_LEVELS x DSG_RECENT_LEN)
for w in ${WORKLOADS:-C2 C3 C4}; do
  for rl in ${LEVELS:-1 2 3 4 6}; do
    for ln in ${LENS:-16 32}; do
      echo -n "$w levels=$rl len=$ln: "
      DSG_RECENT_LEVELS=$rl DSG_RECENT_LEN=$ln python tools/profile_one.py $w 3 | sed -e "s/.*'t_dp_ms': \([0-9.]*\).*/dp_ms \1/"
    done
  done
done
