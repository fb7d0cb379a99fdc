timeout 300 bash tools/knob_bench.sh C1 "DSG_RUNNERS=24" "DSG_RUNNERS=32" "DSG_GRADE1=2" "DSG_GRADE1=5" "DSG_FIN_FOLD=8" "DSG_FIN_FOLD=64" "DSG_CHUNK_LEN1=32"
timeout 300 bash tools/knob_bench.sh C4 "DSG_RUNNERS=24" "DSG_RUNNERS=20"
timeout 300 bash tools/knob_bench.sh C2 "DSG_RUNNERS=24"
