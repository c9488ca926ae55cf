# round-2 GPU job 34: short-walk shape threshold on the L2-resident cfg3 (the short shape is issue-bound there)
set -x
O=gpurun_out
for t in 20 0 8 12 20 0; do
  echo "== cfg3 SABA_SHORT_STEPS=$t" >> $O/r02ah_short.txt
  SABA_SHORT_STEPS=$t python tools/aesc_run.py --workload cfg3 --reps 2 2>/dev/null | grep "aesc:" >> $O/r02ah_short.txt
done
cat $O/r02ah_short.txt
