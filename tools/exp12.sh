python -m pytest tests -m gpu -x -q > gpurun_out/exp12_tests.log 2>&1
SABA_TRACE=1 python tools/aesc_run.py --workload cfg5 --sources 256 --reps 2 > gpurun_out/exp12_cfg5.log 2>&1
python bench.py --workload cfg3 --no-cpu-baseline > gpurun_out/exp12_cfg3.json 2>&1
