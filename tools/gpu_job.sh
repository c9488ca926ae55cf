# round-2 GPU job 24: u32 global counters in the rank kernel (c32=1), cost of the 16-bit counters' barrier (nosync build: timing only)
set -x
O=gpurun_out
for w in "" "c32=1" "" "c32=1"; do
  echo "== cfg2 [$w]" >> $O/r02x_k2.txt
  SABA_WALK_VARIANT=$w python tools/profile_campaign.py --reps 3 2>&1 | tail -2 >> $O/r02x_k2.txt
done
export SABA_LIB=$PWD/paper_2410_14056_b200/_variants/nosync/libsaba_cuda.so
echo "== cfg2 nosync build" >> $O/r02x_k2.txt
python tools/profile_campaign.py --reps 3 2>&1 | tail -2 >> $O/r02x_k2.txt
echo "== cfg1 nosync build" >> $O/r02x_k2.txt
python tools/profile_campaign.py --workload cfg1 --reps 3 2>&1 | tail -2 >> $O/r02x_k2.txt
unset SABA_LIB
echo "== cfg1" >> $O/r02x_k2.txt
python tools/profile_campaign.py --workload cfg1 --reps 3 2>&1 | tail -2 >> $O/r02x_k2.txt
cat $O/r02x_k2.txt
python -m pytest tests/test_variants_gpu.py -m gpu -x -q -p no:cacheprovider -k campaign > $O/r02x_pytest.log 2>&1; tail -3 $O/r02x_pytest.log
