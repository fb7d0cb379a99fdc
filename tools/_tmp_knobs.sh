DSG_TRACE_FILE=gpurun_out/c4_trace_st2.bin python tools/profile_one.py C4 2
for w in C4 C1 C2 C3 "C5:16,1,1,300"; do bash tools/knob_bench.sh $w "DSG_FIN_POLL_NS=0"; done
