python -m pytest tests/test_parity_gpu.py tests/test_virtual_shards_gpu.py tests/test_edges_gpu.py tests/test_reference_suites_gpu.py tests/test_dpl.py -m gpu -q -x 2>&1 | tail -2
for w in C1 C2; do DSG_PREP_TRACE=1 python tools/host_marks.py $w 5 2>&1 | tail -11 | grep "host\|device"; done
bash tools/gpu_check.sh "" "C1 C4 C2" plan
