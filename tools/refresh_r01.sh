# Round-1 refresh of the committed measurements (run under gpurun).
python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/rf_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rf_smoke.log 2>&1
python bench.py > gpurun_out/rf_bench_cfg2.json 2> gpurun_out/rf_bench_cfg2.err
python bench.py --workload cfg1 --no-aesc > gpurun_out/rf_bench_cfg1.json 2> gpurun_out/rf_bench_cfg1.err
python bench.py --workload cfg3 > gpurun_out/rf_bench_cfg3.json 2> gpurun_out/rf_bench_cfg3.err
python bench.py --workload cfg5 > gpurun_out/rf_bench_cfg5.json 2> gpurun_out/rf_bench_cfg5.err
python bench.py --workload cfg4 --no-cpu-baseline > gpurun_out/rf_bench_cfg4.json 2> gpurun_out/rf_bench_cfg4.err
python tests/qa/graph_build_bench.py > gpurun_out/rf_graph_build.txt 2>&1
SABA_TRACE=1 python tools/e2e_trace_cfg3.py > gpurun_out/rf_e2e_trace.log 2>&1
python bench.py --impl reference > gpurun_out/rf_bench_reference_arm.json 2> gpurun_out/rf_bench_reference_arm.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rf_launches_cfg2.csv python bench.py --steps 2 --warmup 1 --no-aesc --no-cpu-baseline > /dev/null 2>&1
