# round-2 GPU job 3: tests, checked build on the protocol cases, REC variant timing
set -x
O=gpurun_out
python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/r02c_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r02c_pytest.log
tail -3 $O/r02c_pytest.log
CHK=$PWD/paper_2410_14056_b200/_variants/checked/libsaba_cuda.so
SABA_LIB=$CHK timeout 900 python tools/sanitize_cases.py > $O/r02c_checked_cases.log 2>&1; echo "rc=$?" >> $O/r02c_checked_cases.log
SABA_LIB=$CHK SABA_WALK_VARIANT=fat=0,hot=1 timeout 900 python tools/sanitize_cases.py >> $O/r02c_checked_cases.log 2>&1; echo "rc=$?" >> $O/r02c_checked_cases.log
SABA_LIB=$CHK SABA_AESC_REC=2 timeout 900 python tools/sanitize_cases.py >> $O/r02c_checked_cases.log 2>&1; echo "rc=$?" >> $O/r02c_checked_cases.log
SABA_LIB=$CHK timeout 1800 python -m pytest tests/test_variants_gpu.py tests/test_multidevice_gpu.py tests/test_aesc_gpu.py tests/test_walks_gpu.py -x -q -p no:cacheprovider -k "not full_size and not cfg" > $O/r02c_checked_pytest.log 2>&1; echo "rc=$?" >> $O/r02c_checked_pytest.log
tail -3 $O/r02c_checked_cases.log $O/r02c_checked_pytest.log
for v in 1 0; do SABA_AESC_REC=$v python tools/aesc_run.py --workload cfg4 --sources 64 --reps 2 > $O/r02c_cfg4_rec$v.log 2>&1; tail -2 $O/r02c_cfg4_rec$v.log; done
for v in 1 2; do SABA_AESC_REC=$v python tools/aesc_run.py --workload cfg5 --sources 512 --reps 2 > $O/r02c_cfg5_rec$v.log 2>&1; tail -2 $O/r02c_cfg5_rec$v.log; done
for v in 1 2; do SABA_AESC_REC=$v python tools/aesc_run.py --workload cfg3 --reps 2 > $O/r02c_cfg3_rec$v.log 2>&1; tail -2 $O/r02c_cfg3_rec$v.log; done
