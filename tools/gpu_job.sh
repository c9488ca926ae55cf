# round-2 GPU job 33: final build — full GPU suite, smoke, default bench + reference arm
set -x
O=gpurun_out
python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/r02ag_pytest_gpu.log 2>&1; echo "rc=$?" >> $O/r02ag_pytest_gpu.log; tail -4 $O/r02ag_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/r02ag_smoke.log 2>&1; tail -2 $O/r02ag_smoke.log
python bench.py --impl reference > $O/r02ag_bench_reference_arm.json 2> $O/r02ag_bench_reference_arm.err
python bench.py > $O/r02ag_bench_default.json 2> $O/r02ag_bench_default.err; tail -c 300 $O/r02ag_bench_default.json
