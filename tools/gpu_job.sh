# round-2 GPU job 27: e2e phase breakdown on cfg1 (small graph: fixed overheads)
set -x
O=gpurun_out
SABA_TRACE=1 python tools/e2e_breakdown.py cfg1 > $O/r02aa_e2e_cfg1.txt 2>&1; grep -v graph_build $O/r02aa_e2e_cfg1.txt | tail -40
