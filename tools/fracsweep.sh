#!/bin/bash
# t_dp_ms for the critical/background CTA split fractions
for f in 0 0.125 0.25 0.4; do
  for w in C2 C4 C1; do
    echo -n "frac=$f $w "; DSG_CRIT_FRAC=$f python tools/profile_one.py $w 3 | python -c "import sys,ast; l=sys.stdin.read(); d=ast.literal_eval(l[l.index('{'):]); print(d['t_dp_ms'], d['t_device_ms'])"
  done
done
