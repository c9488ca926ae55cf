python -m pytest tests/test_aesc_gpu.py -x -q > gpurun_out/exp7_tests.log 2>&1
bash tools/exp_variants.sh gpurun_out/exp7.log main grab4 grab32
SABA_AESC_WORKERS=1 python tools/aesc_run.py --workload cfg3 --reps 2 2>&1 | grep aesc: >> gpurun_out/exp7.log
