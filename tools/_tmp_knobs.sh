timeout 600 bash tools/knob_bench.sh C4 "DSG_GRADE1=5" "DSG_GRADE1=6" "DSG_GRADE1=8"
for w in C1 C2 C3 "C5:8,2,7,600" "C5:16,1,1,300"; do timeout 300 bash tools/knob_bench.sh $w "DSG_GRADE1=5" "DSG_GRADE1=6"; done
