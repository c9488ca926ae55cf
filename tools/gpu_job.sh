set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02a_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02a_pytest.log
tail -5 gpurun_out/r02a_pytest.log
python bench.py --steps 5 --warmup 3 --no-aesc > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err; echo bench rc=$?
tail -c 3000 gpurun_out/r02a_bench.json
