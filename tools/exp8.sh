python -m pytest tests/test_aesc_gpu.py -x -q > gpurun_out/exp8_tests.log 2>&1
bash tools/exp_variants.sh gpurun_out/exp8.log main
SABA_AESC_WORKERS=1 python tools/aesc_run.py --workload cfg3 --reps 2 2>&1 | grep aesc: >> gpurun_out/exp8.log
SABA_AESC_WORKERS=1 python tools/aesc_run.py --workload cfg4 --sources 64 --reps 2 2>&1 | grep aesc: >> gpurun_out/exp8.log
