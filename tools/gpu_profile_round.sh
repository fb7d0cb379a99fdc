#!/bin/bash
# Round-end evidence: bench lines, reference arm, launch list and one full
# ncu capture of the DP kernel (run under gpurun; outputs in gpurun_out/).
mkdir -p gpurun_out
timeout 300 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench.err
for w in C1 C3 C4 C5:8,2,7,600; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 10 > gpurun_out/bench_${w%%:*}.json 2>> gpurun_out/bench.err
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:persistent_levels -s 2 -c 1 \
  -o gpurun_out/c2_full python tools/profile_one.py C2 3 > gpurun_out/ncu_full.log 2>&1
