python -m pytest tests/test_graph_build_gpu.py -x -q > gpurun_out/exp13_tests.log 2>&1
python bench.py --steps 5 > gpurun_out/exp13_cfg2.json 2> gpurun_out/exp13_cfg2.err
python bench.py --workload cfg3 --no-cpu-baseline > gpurun_out/exp13_cfg3.json 2> gpurun_out/exp13_cfg3.err
python bench.py --workload cfg5 --no-cpu-baseline --steps 1 --warmup 1 > gpurun_out/exp13_cfg5.json 2> gpurun_out/exp13_cfg5.err
