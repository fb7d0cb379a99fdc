#!/bin/bash
# Round-end evidence: bench lines (device + e2e + CPU baseline) for every
# workload and variant, the reference arm, the GPU test suite and smoke.
#   gpurun -- bash tools/final_bench.sh TAG
TAG=${1:-r2}
OUT=gpurun_out/final_${TAG}
mkdir -p $OUT
for w in C2 C1 C3 C4 "C5:8,2,7,600" "C5:16,1,1,300" "C5:8,2,7,1900" "C5:16,1,1,1300" C2@seed2 C2@D1000 C2@int64; do
  f=${w//[:,@]/_}
  timeout 600 python bench.py --workload "$w" > $OUT/bench_$f.json 2> $OUT/bench_$f.err
  echo "$w rc=$? $(tail -c 300 $OUT/bench_$f.json | head -c 0)"
done
timeout 600 python bench.py --impl reference > $OUT/bench_reference.json 2> $OUT/bench_reference.err
echo "reference rc=$?"
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
echo "default rc=$?"
timeout 1500 python -m pytest tests -m gpu -q > $OUT/gpu_tests.log 2>&1
echo "gpu tests rc=$?"; tail -2 $OUT/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > $OUT/smoke.log 2>&1
echo "smoke rc=$?"; tail -2 $OUT/smoke.log
