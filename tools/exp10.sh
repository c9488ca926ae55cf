python -m pytest tests/test_aesc_gpu.py -x -q > gpurun_out/exp10_tests.log 2>&1
for v in main pb3 pb4u4; do
  if [ $v = main ]; then unset SABA_LIB; else export SABA_LIB=$PWD/paper_2410_14056_b200/_variants/$v/libsaba_cuda.so; fi
  echo "== $v" >> gpurun_out/exp10.log
  SABA_AESC_WORKERS=1 python tools/aesc_run.py --workload cfg3 --reps 2 2>&1 | grep aesc: >> gpurun_out/exp10.log
  python tools/aesc_run.py --workload cfg3 --reps 2 2>&1 | grep aesc: >> gpurun_out/exp10.log
  python tools/aesc_run.py --workload cfg4 --sources 64 --reps 2 2>&1 | grep aesc: >> gpurun_out/exp10.log
done
