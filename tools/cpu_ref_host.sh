#!/bin/bash
# Full-size reference CPU solves on the GPU box's host (one process per
# workload group, each single-threaded), with the host description.
#   gpurun -- bash tools/cpu_ref_host.sh
set -u
mkdir -p gpurun_out/cpu_ref
D=gpurun_out/cpu_ref
{ lscpu; echo; nproc; echo; uptime; free -g; } > $D/lscpu.txt 2>&1
python -c "import __graft_entry__" 2>/dev/null
pids=()
run() { local tag=$1; shift; python tools/cpu_ref_host.py $D/$tag.json "$@" > $D/$tag.log 2>&1 & pids+=($!); }
run c2 C2
run c5top C5:8,2,7,600
run c2seed2 C2@seed2
run c2d1000 C2@D1000
run c3 C3
run sparse C5:16,1,1,300
run small C1 C4
for p in "${pids[@]}"; do wait $p; done
uptime >> $D/lscpu.txt
echo CPU_REF_DONE
