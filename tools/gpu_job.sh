# round-2 GPU job 29: aesc_walk_hub (hub rho in shared memory, tile hand-out) — parity and cfg3 timing by hub count
set -x
O=gpurun_out
python -m pytest tests/test_aesc_gpu.py tests/test_variants_gpu.py tests/test_fullsize_reference_gpu.py -m gpu -x -q -p no:cacheprovider -k "aesc or cfg3" > $O/r02ac_pytest.log 2>&1; echo "rc=$?" >> $O/r02ac_pytest.log; tail -4 $O/r02ac_pytest.log
for h in 0 12288 4096 8192 16383 0 12288; do
  echo "== cfg3 HUB=$h" >> $O/r02ac_hub.txt
  SABA_AESC_HUB=$h python tools/aesc_run.py --workload cfg3 --reps 2 2>/dev/null | grep "aesc:" >> $O/r02ac_hub.txt
done
for h in 0 12288; do
  echo "== cfg3 HUB=$h workers=1" >> $O/r02ac_hub.txt
  SABA_AESC_WORKERS=1 SABA_AESC_HUB=$h python tools/aesc_run.py --workload cfg3 --reps 2 2>/dev/null | grep "aesc:" >> $O/r02ac_hub.txt
done
cat $O/r02ac_hub.txt
