# round-2 GPU job 38: propagation depths per CUDA-graph replay on cfg3 (default 8)
set -x
O=gpurun_out
for d in 8 16 32 8 16; do
  echo "== cfg3 SABA_DEPTHS_PER_GRAPH=$d" >> $O/r02al_depths.txt
  SABA_DEPTHS_PER_GRAPH=$d python tools/aesc_run.py --workload cfg3 --reps 2 2>/dev/null | grep "aesc:" >> $O/r02al_depths.txt
done
cat $O/r02al_depths.txt
