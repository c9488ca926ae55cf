# round-2 GPU job 9: column-sparse pull + rec/l1hot K2 variants
set -x
O=gpurun_out
python -m pytest tests/test_variants_gpu.py -x -q -p no:cacheprovider > $O/r02i_pytest_variants.log 2>&1; echo "rc=$?" >> $O/r02i_pytest_variants.log; tail -3 $O/r02i_pytest_variants.log
for v in -1 0 1; do SABA_PULL_SKIP=$v python tools/aesc_run.py --workload cfg5 --sources 512 --reps 2 > $O/r02i_cfg5_skip$v.log 2>&1; grep "^aesc:" $O/r02i_cfg5_skip$v.log | tail -1; done
for v in -1 0; do SABA_PULL_SKIP=$v python tools/aesc_run.py --workload cfg3 --reps 2 > $O/r02i_cfg3_skip$v.log 2>&1; grep "^aesc:" $O/r02i_cfg3_skip$v.log | tail -1; done
for v in -1 0; do SABA_PULL_SKIP=$v python tools/aesc_run.py --workload cfg4 --sources 64 --reps 2 > $O/r02i_cfg4_skip$v.log 2>&1; grep "^aesc:" $O/r02i_cfg4_skip$v.log | tail -1; done
bash tools/sweep_walk.sh "" "rec=1,l1hot=12288" "rec=1,l1hot=4096" "rec=1,l1hot=0" "rec=1,l1hot=24576" "" > $O/r02i_sweep.txt 2>&1; cat $O/r02i_sweep.txt
